#!/bin/bash
# First GPU pass: parity tests, smoke, bench, launch list, one full ncu capture.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
echo "pytest rc=${PIPESTATUS[0]}"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
head -c 4000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rnbp1000.csv \
  python tools/profile_step.py --n 1000 --kind rnbp --iters 200 > /dev/null 2>&1; echo ncu1=$?
python tools/launch_summary.py gpurun_out/launches_rnbp1000.csv 2>&1 | head -20
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_vertex_update -s 5 -c 2 \
  -o gpurun_out/prof_lbp4096 python tools/profile_step.py --n 4096 --kind lbp --iters 6 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ls -la gpurun_out
