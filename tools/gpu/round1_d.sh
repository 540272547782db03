#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=900 bash tools/gpu/run_tests.sh
timeout 900 python tools/configs_probe.py --big --skip-rs --only ising1000,ising4096,ising16k,potts > gpurun_out/probe4.jsonl 2> gpurun_out/probe4.err; echo probe=$?
cat gpurun_out/probe4.jsonl | cut -c1-330; tail -3 gpurun_out/probe4.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_vertex_update -s 5 -c 1 \
  -o gpurun_out/prof_lbp4096_lat3 python tools/profile_step.py --n 4096 --kind lbp --iters 6 > gpurun_out/ncu_lat3.log 2>&1; echo ncu=$?
