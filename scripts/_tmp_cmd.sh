OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
L="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$L > $OUT/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $L > $OUT/ncu.log 2>&1
python scripts/launch_table.py $OUT/launches.csv 2>/dev/null | head -14
python -c "import json; d=json.loads(open('$OUT/plain.log').read().strip().splitlines()[-1]); print(d['phases_ms'], d['value']/1e9)"
