OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pipelined or projection_matches" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log
timeout 600 python bench.py --config 4 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err
python -c "import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print('value %.4e'%d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e'], 'clocks', d['clocks'])"
