set -x
timeout 600 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -25
timeout 600 python bench.py --steps 3 --warmup 1 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?; tail -c 3000 gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rnbp1000.csv python tools/profile_step.py --n 1000 --kind rnbp --iters 30 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_vertex_update -s 3 -c 2 -o gpurun_out/prof_rnbp_update python tools/profile_step.py --n 1000 --kind rnbp --iters 10 > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_vertex_update -s 3 -c 2 -o gpurun_out/prof_lbp4096 python tools/profile_step.py --n 4096 --kind lbp --iters 6 > gpurun_out/ncu3.log 2>&1; echo ncu3=$?
ls -la gpurun_out
