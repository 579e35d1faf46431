#!/bin/bash
# One gpurun call producing a round's measurement record: GPU tests, smoke, the full bench line (C4 + C5/C1-C3
# sub-records, cpu_baseline, e2e), the reference arm, the bench's ncu launch list, and ncu --set full of the step
# kernels at --clock-control none and base. usage (on the box): bash scripts/gpu_record.sh TAG
TAG=${1:-r02rec}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?" >> $OUT/bench_ref.err
L="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-c5 --no-small"
$L > $OUT/plain_launches.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches.csv $L > $OUT/ncu_launches.log 2>&1
K='regex:k_tet_weights|k_assemble_mask|k_block_pcg|k_proj_y|k_proj_ai|k_proj_bg_mma|k_proj_final'
F="python scripts/prof_pcg.py --reps 1 --project"
$F > $OUT/plain_full.log 2>&1 && for cc in none base; do
  timeout 900 ncu --set full --clock-control $cc --import-source on -k "$K" -o $OUT/step_$cc $F > $OUT/ncu_step_$cc.log 2>&1
done
tail -4 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log; tail -1 $OUT/bench.err; tail -1 $OUT/bench_ref.err
python -c 'import json,sys; d=json.loads(open(sys.argv[1]).read()); print(d["value"], d["phases_ms"], d["roofline"]["frac"], d.get("next1_ms"), d["e2e"]["value"], d.get("c5",{}).get("value"))' $OUT/bench.json
ls $OUT
