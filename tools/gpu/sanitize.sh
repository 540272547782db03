#!/bin/bash
# compute-sanitizer passes over a -m gpu subset that reaches every kernel
# family: lattice / CSR / q-state sweeps (fused finalize), RnBP graph loop and
# persistent tail, RBP radix select, RS splashes (cooperative), band halos,
# the collapse-checked log-domain path.  memcheck and synccheck run the whole
# subset in one process; racecheck runs one test per process on the
# non-cooperative kernels (it cannot run grid-synchronising cooperative
# launches: the process faults inside the tool).  Logs: gpurun_out/sanitize_*.log
set -u
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SUB="tests/test_gpu_parity.py::test_lbp_lockstep_ising_binary tests/test_gpu_parity.py::test_lbp_lockstep_random_generic \
 tests/test_gpu_parity.py::test_rnbp_injected_frontier_lockstep tests/test_gpu_parity.py::test_rbp_topk_exact_against_select_top_k \
 tests/test_gpu_parity.py::test_zero_edge_graph tests/test_gpu_parity.py::test_tree_exactness_all_device_schedulers \
 tests/test_gpu_splash.py::test_splash_apply_lockstep_with_reference_splashes tests/test_gpu_splash.py::test_rs_run_tree_exact \
 tests/test_gpu_lbp_sweeps.py::test_tma_sweep_lockstep_descriptor_lattices \
 tests/test_gpu_parallel.py::test_band_lbp_bitwise_equals_unpartitioned tests/test_gpu_numeric.py \
 tests/test_gpu_parity.py::test_rnbp_persistent_tail_matches_graph_loop \
 tests/test_gpu_fused.py::test_fused_run_equals_two_launch_loop tests/test_gpu_fused.py::test_fused_empty_frontier_hands_the_iteration_back \
 tests/test_gpu_parallel.py::test_parts_rnbp_fallback_across_parts tests/test_gpu_parallel.py::test_parts_generic_binary_tables_and_lattices"
for tool in memcheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -p no:cacheprovider $SUB > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
: > gpurun_out/sanitize_racecheck.log
for t in tests/test_gpu_parity.py::test_lbp_lockstep_ising_binary tests/test_gpu_parity.py::test_lbp_lockstep_random_generic \
         tests/test_gpu_parity.py::test_rbp_topk_exact_against_select_top_k \
         "tests/test_gpu_lbp_sweeps.py::test_tma_sweep_lockstep_descriptor_lattices[7-1030]" \
         "tests/test_gpu_lbp_sweeps.py::test_tiles_sweep_lockstep_descriptor_lattices[5-1537]" \
         tests/test_gpu_lbp_sweeps.py::test_potts_lattice_sweep_lockstep tests/test_gpu_splash.py::test_splash_apply_lockstep_with_reference_splashes \
         "tests/test_gpu_parallel.py::test_band_lbp_bitwise_equals_unpartitioned[2]" \
         "tests/test_gpu_numeric.py::test_collapse_at_the_first_refresh[lbp]" \
         "tests/test_gpu_numeric.py::test_flagged_model_without_collapse_matches_reference[rbp]" \
         "tests/test_gpu_fused.py::test_fused_run_equals_two_launch_loop[30-2.5-1-0.5]" \
         "tests/test_gpu_parallel.py::test_parts_lbp_random_graph_bitwise_equals_unpartitioned[3]"; do
  echo "== $t" >> gpurun_out/sanitize_racecheck.log
  timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 --print-limit 10 \
      python -m pytest -q -p no:cacheprovider "$t" >> gpurun_out/sanitize_racecheck.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
done
