#!/bin/bash
# Round-2 final evidence: ncu --set full of the fused RnBP sweep at 1000^2
# (headline kernel, per-warp tiles) and of the RBP top-k list kernels; the
# launch list of the bench command.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
P="python tools/profile_step.py"
timeout 600 $NCU -k regex:k_rnbp_fused -s 6 -c 1 -o gpurun_out/r2g_fused1000 $P --n 1000 --kind rnbp --iters 10 > /dev/null 2>&1; echo fused1000=$?
timeout 600 $NCU -k regex:"k_rx_|k_rbp_commit_list" -s 12 -c 5 -o gpurun_out/r2g_rbp_topk $P --n 1000 --kind rbp --iters 6 > /dev/null 2>&1; echo topk=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r2g_launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2g_bench_under_ncu.log 2>&1; echo launches=$?
ls -la gpurun_out/r2g_*
