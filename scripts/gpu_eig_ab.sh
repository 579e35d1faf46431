#!/bin/bash
# A/B of the filtered pencil eigensolver's knobs on one box: bash scripts/gpu_eig_ab.sh TAG "ENV1" "ENV2" ...
# (each ENV a space-separated NAME=VALUE list, "" = defaults): event/wall time per call and rounds per variant at C4
# and C5, then the NEXT-1/2 and lifecycle tests.
TAG=${1:-eigab}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
for c in 4 5; do
  for v in "$@"; do
    echo "== C$c [$v]" >> $OUT/eig.log
    env $v KS_EF_VERBOSE=1 timeout 300 python scripts/prof_eig.py --config $c --reps 1 2>&1 | grep "round" | tail -1 >> $OUT/eig.log
    env $v timeout 300 python scripts/prof_eig.py --config $c --reps 6 2>&1 | grep pencil_eig | tail -4 >> $OUT/eig.log
  done
done
timeout 900 python -m pytest tests/test_gpu_next1.py tests/test_gpu_next2.py tests/test_gpu_lifecycle.py -x -q > $OUT/pytest_next.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_next.log
cat $OUT/eig.log; tail -3 $OUT/pytest_next.log
