#!/bin/bash
# compute-sanitizer passes (memcheck / racecheck / synccheck) over a small -m gpu
# subset that reaches every kernel family: lattice + CSR + q-state sweeps, RnBP
# graph loop and persistent tail, RBP radix select, RS splashes, band halos.
# Output: gpurun_out/sanitize_<tool>.log (summaries under profiles/).
set -u
mkdir -p gpurun_out
SUB="tests/test_gpu_parity.py::test_lbp_lockstep_ising_binary tests/test_gpu_parity.py::test_lbp_lockstep_random_generic \
 tests/test_gpu_parity.py::test_rnbp_injected_frontier_lockstep tests/test_gpu_parity.py::test_rbp_topk_exact_against_select_top_k \
 tests/test_gpu_parity.py::test_zero_edge_graph tests/test_gpu_parity.py::test_tree_exactness_all_device_schedulers \
 tests/test_gpu_splash.py::test_splash_apply_lockstep_with_reference_splashes tests/test_gpu_splash.py::test_rs_run_tree_exact \
 tests/test_gpu_lbp_sweeps.py::test_tma_sweep_lockstep_descriptor_lattices \
 tests/test_gpu_parallel.py::test_band_lbp_bitwise_equals_unpartitioned tests/test_gpu_numeric.py"
PERSIST="tests/test_gpu_parity.py::test_rnbp_persistent_tail_matches_graph_loop"
for tool in memcheck racecheck synccheck; do
  sel="$SUB"
  [ "$tool" = memcheck ] && sel="$SUB $PERSIST"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -p no:cacheprovider -x $sel > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
