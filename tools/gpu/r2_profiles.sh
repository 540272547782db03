#!/bin/bash
# Round-2 evidence: ncu launch list of the bench command and one --set full
# capture per dominant kernel (digested into profiles/ by tools/ncu_digest.py).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2_bench_under_ncu.log 2>&1; echo launches=$?
P="python tools/profile_step.py"
timeout 600 $NCU -k regex:k_rnbp_select -s 5 -c 1 -o gpurun_out/r2_prof_select $P --n 1000 --kind rnbp --iters 20 > /dev/null 2>&1; echo select=$?
timeout 600 $NCU -k regex:k_vertex_update -s 6 -c 1 -o gpurun_out/r2_prof_refresh $P --n 1000 --kind rnbp --iters 20 > /dev/null 2>&1; echo refresh=$?
timeout 600 $NCU -k regex:k_lbp_lattice -s 2 -c 1 -o gpurun_out/r2_prof_lbp16k $P --n 16384 --kind lbp --iters 3 > /dev/null 2>&1; echo lbp16k=$?
timeout 600 $NCU -k regex:k_vertex_update -s 4 -c 1 -o gpurun_out/r2_prof_lbp1000 $P --n 1000 --kind lbp --iters 6 > /dev/null 2>&1; echo lbp1000=$?
timeout 600 $NCU -k regex:k_vertex_update -s 2 -c 1 -o gpurun_out/r2_prof_potts $P --n 4096 --potts 8 --kind lbp --iters 3 > /dev/null 2>&1; echo potts=$?
timeout 600 $NCU -k regex:k_rnbp_persist -c 1 -o gpurun_out/r2_prof_persist python tools/rnbp_trace.py 1000 > /dev/null 2>&1; echo persist=$?
timeout 600 $NCU -k regex:k_rs_iteration -s 1 -c 1 -o gpurun_out/r2_prof_rs $P --n 1000000 --er --kind rs --iters 3 > /dev/null 2>&1; echo rs=$?
timeout 600 $NCU -k regex:k_rx_compact -s 3 -c 1 -o gpurun_out/r2_prof_radix $P --n 1000 --kind rbp --iters 3 > /dev/null 2>&1; echo radix=$?
ls -la gpurun_out/*.ncu-rep
