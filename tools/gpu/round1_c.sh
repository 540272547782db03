#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=900 bash tools/gpu/run_tests.sh
timeout 900 python tools/configs_probe.py --big --skip-rs > gpurun_out/probe3.jsonl 2> gpurun_out/probe3.err; echo probe=$?
cat gpurun_out/probe3.jsonl; tail -3 gpurun_out/probe3.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_vertex_update -s 5 -c 1 \
  -o gpurun_out/prof_lbp4096_lat2 python tools/profile_step.py --n 4096 --kind lbp --iters 6 > gpurun_out/ncu_lat2.log 2>&1; echo ncu=$?
