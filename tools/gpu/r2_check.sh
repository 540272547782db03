#!/bin/bash
# Round-2 full check: every -m gpu test (no -x, so all failures show), smoke, one bench line.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputests.log 2>&1; echo tests_rc=$?
tail -30 gpurun_out/r2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r2_bench.json; tail -5 gpurun_out/r2_bench.err
