OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
F="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$F > $OUT/plain_full.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:$2" -s 4 -c 3 -o $OUT/full $F > $OUT/ncu_full.log 2>&1
tail -3 $OUT/ncu_full.log
