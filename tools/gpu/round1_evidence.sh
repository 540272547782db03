#!/bin/bash
# Bench line + ncu launch list of the bench command + full captures of the
# dominant kernels (persistent RnBP tail on 1000^2, LBP sweep on 16384^2).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/bench_under_ncu.log 2>&1; echo ncu_launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rnbp_persist -c 1 \
  -o gpurun_out/prof_persist_final python tools/rnbp_trace.py 1000 > gpurun_out/ncu_persist.log 2>&1; echo ncu_persist=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lbp_lattice -s 2 -c 1 \
  -o gpurun_out/prof_lbp16k_final python tools/profile_step.py --n 16384 --kind lbp --iters 3 > gpurun_out/ncu_lbp.log 2>&1; echo ncu_lbp=$?
