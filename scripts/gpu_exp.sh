#!/bin/bash
# Node-ordering experiment: scripts/exp_order.py with the gathered and the staged S phase.
# usage (on the box): bash scripts/gpu_exp.sh TAG
OUT=gpurun_out/$1; shift
mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
KS_PCG_STAGE=0 timeout 600 python scripts/exp_order.py 4 lex,morton,block4,block8 > $OUT/order_unstaged.jsonl 2> $OUT/order_unstaged.err
KS_PCG_STAGE=1 timeout 600 python scripts/exp_order.py 4 lex,morton,block8 > $OUT/order_staged.jsonl 2> $OUT/order_staged.err
cat $OUT/*.jsonl
