OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_next2.py tests/test_gpu_next1.py tests/test_gpu_next3.py -x -q --durations=5 > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
tail -25 $OUT/pytest.log
