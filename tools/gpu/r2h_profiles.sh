#!/bin/bash
# Round-2 (late) evidence: the bench line after the q-vector select change, and
# ncu --set full of the Potts 4096^2 q=8 RnBP select (quad commits) and touched
# refresh in a dense iteration.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo bench=$?
NCU="ncu --set full --import-source on --clock-control none"
P="python tools/profile_step.py"
timeout 600 $NCU -k regex:k_rnbp_select -s 1 -c 1 -o gpurun_out/r2h_qselect $P --n 4096 --potts 8 --kind rnbp --iters 4 > /dev/null 2>&1; echo qselect=$?
timeout 600 $NCU -k regex:k_lattice_qsweep -s 1 -c 1 -o gpurun_out/r2h_qrefresh $P --n 4096 --potts 8 --kind rnbp --iters 4 > /dev/null 2>&1; echo qrefresh=$?
ls -la gpurun_out/r2h_*
