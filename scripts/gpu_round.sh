#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (full line), ncu launch list, ncu --set full of the top kernels.
# usage (on the box): bash scripts/gpu_round.sh TAG [CONFIG]
TAG=${1:-r01}
CFG=${2:-4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 900 python bench.py --config 5 --steps 5 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 exit $?" >> $OUT/bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?" >> $OUT/bench_ref.err
L="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$L > $OUT/plain_launches.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv $L > $OUT/ncu_launches.log 2>&1
F="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$F > $OUT/plain_full.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_block_pcg|k_proj_a|k_proj_bg|k_proj_y|k_assemble_rows' -s 16 -c 5 -o $OUT/full $F > $OUT/ncu_full.log 2>&1
tail -12 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/bench.json $OUT/bench_c5.json $OUT/bench_ref.json
ls -la $OUT
