OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
KS_PCG_STAGE=1 timeout 600 python scripts/exp_order.py 4 lex,morton,block8,block4 > $OUT/order_stage1.jsonl 2>&1
KS_PCG_STAGE=0 timeout 600 python scripts/exp_order.py 4 morton,block8 > $OUT/order_stage0.jsonl 2>&1
cat $OUT/*.jsonl
