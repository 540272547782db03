#!/bin/bash
# Round-2 evidence: ncu --set full of the fused RnBP sweep (headline 1000^2 and
# config 5 16384^2), the q-state lanes sweep, the LBP sweeps; the launch list of
# the bench command; compute-sanitizer over a -m gpu subset.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
P="python tools/profile_step.py"
timeout 600 $NCU -k regex:k_rnbp_fused -s 6 -c 1 -o gpurun_out/r2e_fused1000 $P --n 1000 --kind rnbp --iters 10 > /dev/null 2>&1; echo fused1000=$?
timeout 900 $NCU -k regex:k_rnbp_fused -s 2 -c 1 -o gpurun_out/r2e_fused16k $P --n 16384 --kind rnbp --iters 4 > /dev/null 2>&1; echo fused16k=$?
timeout 600 $NCU -k regex:k_lbp_lattice -s 2 -c 1 -o gpurun_out/r2e_lbp16k $P --n 16384 --kind lbp --iters 3 > /dev/null 2>&1; echo lbp16k=$?
timeout 600 $NCU -k regex:k_lattice_qsweep -s 2 -c 1 -o gpurun_out/r2e_qsweep $P --n 4096 --potts 8 --kind lbp --iters 3 > /dev/null 2>&1; echo qsweep=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r2e_launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2e_bench_under_ncu.log 2>&1; echo launches=$?
timeout 2400 bash tools/gpu/sanitize.sh; echo sanitize=$?
for t in memcheck synccheck racecheck; do echo "== $t"; grep -E "ERROR SUMMARY|rc=|passed|failed" gpurun_out/sanitize_$t.log | tail -14; done
