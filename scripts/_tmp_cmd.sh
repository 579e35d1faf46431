OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
timeout 900 python scripts/scf_demo.py 48 10 20 > $OUT/scf_48_mu20.json 2> $OUT/scf1.err

timeout 900 python scripts/scf_demo.py 48 10 1600 > $OUT/scf_48_mu1600.json 2> $OUT/scf3.err
for f in $OUT/*.json; do cat $f; echo; done; for f in $OUT/*.err; do tail -3 $f; done
