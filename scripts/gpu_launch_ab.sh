#!/bin/bash
# Launch-list A/B of libks variants: bash scripts/gpu_launch_ab.sh TAG [pytest]
OUT=gpurun_out/$1; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
if [ "$2" == "pytest" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
fi
L="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
for v in default paper_2404_19249_b200/libks_*.so; do
  n=$(basename $v .so)
  if [ "$v" == "default" ]; then unset KS_LIB; else export KS_LIB=$PWD/$v; fi
  $L > $OUT/plain_$n.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$n.csv $L > $OUT/ncu_$n.log 2>&1
  echo "=== $n"; python scripts/launch_table.py $OUT/launches_$n.csv 2>/dev/null | grep -v "cub::\|k_stiff\|k_emap\|k_item\|k_slotmap\|k_inv_ptr\|k_pair\|k_geom\|k_cols\|k_row_ptr\|k_local\|k_sell\|k_diag\|k_check\|k_notdir\|k_free\|k_P_rows\|k_group\|k_lower\|k_pv4\|at::" | head -12
  python -c "import json; d=json.loads(open('$OUT/plain_$n.log').read().strip().splitlines()[-1]); print(d['phases_ms'], d['value']/1e9)"
done
unset KS_LIB
