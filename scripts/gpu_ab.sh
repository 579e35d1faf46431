#!/bin/bash
# A/B of libks variants on one box: bash scripts/gpu_ab.sh TAG [pytest]
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1
if [ "$2" == "pytest" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
B="python bench.py --config 4 --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 $B > $OUT/bench_default.json 2> $OUT/bench_default.err
for v in paper_2404_19249_b200/libks_*.so; do
  n=$(basename $v .so)
  KS_LIB=$PWD/$v timeout 300 $B > $OUT/bench_$n.json 2> $OUT/bench_$n.err
done
KS_SPMM_VARIANT=0 timeout 300 python scripts/exp_spmm.py 4 8,16,32 > $OUT/spmm.jsonl 2>&1
cat $OUT/spmm.jsonl
for f in $OUT/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ph = d.get("pcg_phases") or {}
    print(f.split("/")[-1], "solve %.3f ms" % d["phases_ms"]["block_solve"], "frac %.3f" % d["roofline"]["frac"],
          " ".join("%s %.1fus %.0fGB/s" % (k, 1e3 * ph[k]["ms"], ph[k]["GB/s"]) for k in ("S", "U", "P") if k in ph),
          "init %.0fus" % (1e3 * ph.get("init_ms", 0)))
except Exception as ex:
    print(f, "failed", ex, open(f.replace(".json", ".err")).read()[-600:])
PY
done
