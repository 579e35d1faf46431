bash scripts/gpu_ab.sh r01h
timeout 600 python scripts/exp_order.py 4 lex,morton,block8 > gpurun_out/r01h/order.jsonl 2>&1; cat gpurun_out/r01h/order.jsonl
