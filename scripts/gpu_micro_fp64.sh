#!/bin/bash
# FP64 pipe microbenchmark + the NEXT-1/2 tests + eigensolver timing: bash scripts/gpu_micro_fp64.sh TAG
TAG=${1:-fp64}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma_peak scripts/micro/dfma_peak.cu && /tmp/dfma_peak > $OUT/dfma_peak.jsonl 2>&1
cat $OUT/dfma_peak.jsonl
for c in 4 5; do for v in "" "KS_EF_GEMM=cublas KS_EF_RR=cublas"; do
  echo "== C$c [$v]" >> $OUT/eig.log
  env $v timeout 300 python scripts/prof_eig.py --config $c --reps 6 2>&1 | grep pencil_eig | tail -4 >> $OUT/eig.log
done; done
cat $OUT/eig.log
timeout 900 python -m pytest tests/test_gpu_next1.py tests/test_gpu_next2.py tests/test_gpu_lifecycle.py -x -q > $OUT/pytest_next.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_next.log
tail -3 $OUT/pytest_next.log
