#!/bin/bash
# GPU parity tests (+ optional extra pytest args), output under gpurun_out/
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout ${T:-900} python -m pytest tests/ -m gpu -q -x "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
