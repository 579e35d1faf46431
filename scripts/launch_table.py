#!/usr/bin/env python
"""Aggregate an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv) by kernel name.
usage: python scripts/launch_table.py launches.csv [skip_first_n_launches]"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = OrderedDict()
for r in rows[i + 1:][skip:]:
    if len(r) <= mi:
        continue
    name = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")[:50]
    v = float(r[mi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    agg.setdefault(name, []).append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} n={len(v):4d} mean={sum(v) / len(v):9.1f}us total={sum(v):10.1f}us {100 * sum(v) / tot:5.1f}%")
