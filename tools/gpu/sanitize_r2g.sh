#!/bin/bash
# compute-sanitizer over the last round-2 additions: RBP top-k list kernels
# (ties across chunks), the persistent dense launch (cluster + grid), deep
# splashes, the band driver's device-side parking (fallback across bands);
# memcheck + synccheck + racecheck, one process each.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SUB="tests/test_gpu_parity.py::test_rbp_topk_ties_across_chunks tests/test_gpu_parity.py::test_rbp_topk_exact_against_select_top_k \
 tests/test_gpu_fused.py::test_fused_persistent_windows \
 tests/test_gpu_splash.py::test_deep_rs_frontier_random_graphs \
 tests/test_gpu_parallel.py::test_cpp_driver_rnbp_fallback_across_bands"
for tool in memcheck synccheck racecheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -p no:cacheprovider $SUB > gpurun_out/sanitize3_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize3_$tool.log
  echo "== $tool"; grep -E "ERROR SUMMARY|passed|failed|rc=" gpurun_out/sanitize3_$tool.log | tail -3
done
