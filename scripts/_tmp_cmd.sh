OUT=gpurun_out/$1; TOOL=$2; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
T="python -m pytest tests/test_gpu_parity.py tests/test_gpu_next1.py tests/test_gpu_next2.py -x -q -k 'not config4 and not ragged and not 3 and not scf'"
bash -c "$T" > $OUT/plain.log 2>&1 && timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 --log-file $OUT/sanitizer_$TOOL.log bash -c "$T" > $OUT/run_$TOOL.log 2>&1; echo "exit $?" >> $OUT/run_$TOOL.log
tail -3 $OUT/plain.log; tail -3 $OUT/run_$TOOL.log; tail -5 $OUT/sanitizer_$TOOL.log
