#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=900 bash tools/gpu/run_tests.sh
timeout 600 python tools/configs_probe.py --only er > gpurun_out/probe_er.jsonl 2> gpurun_out/probe_er.err; echo probe=$?
cat gpurun_out/probe_er.jsonl; tail -3 gpurun_out/probe_er.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_vertex_update -s 5 -c 1 \
  -o gpurun_out/prof_lbp4096_lat python tools/profile_step.py --n 4096 --kind lbp --iters 6 > gpurun_out/ncu_lat.log 2>&1; echo ncu=$?
