OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_next1.py tests/test_gpu_next2.py tests/test_gpu_edges.py -x -q > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log
for v in 0 1; do KS_PENCIL_ALL=$v timeout 300 python bench.py --config 4 --steps 5 --no-cpu-baseline --no-e2e > $OUT/b$v.json 2>&1; python -c "import json; d=json.loads(open('$OUT/b$v.json').read().strip().splitlines()[-1]); print('all=$v', d['next1_ms'])"; done
