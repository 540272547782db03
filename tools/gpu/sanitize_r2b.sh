#!/bin/bash
# compute-sanitizer over the round-2 additions: q-state lanes refresh, vertex-range parts,
# .pgm ingest, fused sweeps, config-scale Potts (memcheck + synccheck in one process each)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SUB="tests/test_gpu_lbp_sweeps.py::test_potts_lattice_sweep_lockstep tests/test_gpu_lbp_sweeps.py::test_potts_lbp_run_matches_oracle \
 tests/test_gpu_parallel.py::test_parts_rnbp_fallback_across_parts tests/test_gpu_parallel.py::test_parts_lbp_converges_like_unpartitioned \
 tests/test_pgm.py::test_parsed_model_runs_like_the_arrays tests/test_gpu_fused.py::test_fused_empty_frontier_hands_the_iteration_back \
 tests/test_gpu_rng.py::test_advance_iteration_rekeys_the_draws"
for tool in memcheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -p no:cacheprovider $SUB > gpurun_out/sanitize2_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize2_$tool.log
  echo "== $tool"; grep -E "ERROR SUMMARY|passed|failed|rc=" gpurun_out/sanitize2_$tool.log | tail -3
done
