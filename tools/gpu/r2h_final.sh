#!/bin/bash
# Round-2 final state: GPU tests, smoke, the bench line, the reference arm,
# the launch list of the bench command and ncu --set full of the headline
# kernel (fused RnBP sweep at 1000^2).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1000 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_gputest.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2h_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2h_final_bench.json 2> gpurun_out/r2h_final_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r2h_launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2h_bench_under_ncu.log 2>&1; echo launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rnbp_fused -s 6 -c 1 -o gpurun_out/r2h_fused1000 \
  python tools/profile_step.py --n 1000 --kind rnbp --iters 10 > /dev/null 2>&1; echo fused1000=$?
