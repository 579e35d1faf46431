#!/bin/bash
# ncu --set full of k_sym_gemm (a few launches of one pencil eigensolve): bash scripts/gpu_eig_ncu.sh TAG [CONFIG]
TAG=${1:-eigncu}; CFG=${2:-4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
python scripts/prof_eig.py --config $CFG --reps 1 > $OUT/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sym_gemm -s 30 -c 4 -o $OUT/symgemm_c$CFG python scripts/prof_eig.py --config $CFG --reps 1 > $OUT/ncu.log 2>&1
tail -2 $OUT/plain.log; ls -la $OUT
