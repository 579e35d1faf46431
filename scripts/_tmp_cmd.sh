OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_edges.py -x -q > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
tail -30 $OUT/pytest.log
