#!/bin/bash
# A/B bench of PCG variants on one box: bash scripts/gpu_ab.sh TAG
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
B="python bench.py --config 4 --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 $B > $OUT/bench_default.json 2> $OUT/bench_default.err
KS_PCG_STAGED=0 timeout 300 $B > $OUT/bench_unstaged.json 2> $OUT/bench_unstaged.err
for v in paper_2404_19249_b200/libks_*.so; do
  n=$(basename $v .so)
  KS_LIB=$PWD/$v timeout 300 $B > $OUT/bench_$n.json 2> $OUT/bench_$n.err
done
P="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$P > $OUT/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block_pcg -s 3 -c 1 -o $OUT/full_k_block_pcg $P > $OUT/ncu_full.log 2>&1
for f in $OUT/bench_*.json; do echo "$f $(python -c "import json,sys; d=json.load(open('$f')); print(d['phases_ms'], d['roofline']['frac'])" 2>&1)"; done
