#!/usr/bin/env python
"""One-line-per-kernel summary of an ncu --set full report (run here, no GPU needed):
duration, DRAM bytes (read + write), DRAM throughput %, L1/L2 throughput %, occupancy, registers.
usage: python scripts/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "nsecond": 1e-9}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")}
        for k, name in KEYS.items():
            if k in h:
                v = r[h.index(k)].replace(",", "")
                try:
                    f = float(v) * UNIT.get(units[h.index(k)], 1)
                except ValueError:
                    f = v
                d[name] = f
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
            d["dram_GBs"] = d["dram_bytes"] / d["duration"] / 1e9 if d.get("duration") else None
        res.append(d)
    for d in res:
        print(f"{d['kernel'][:40]:40s} {1e6 * d.get('duration', 0):10.1f} us  DRAM {d.get('dram_bytes', 0) / 1e9:8.3f} GB "
              f"({d.get('dram_GBs') or 0:7.0f} GB/s, {d.get('dram_pct', 0):5.1f}%)  L1 {d.get('l1_pct', 0):5.1f}%  "
              f"L2 {d.get('l2_pct', 0):5.1f}%  occ {d.get('occupancy_pct', 0):5.1f}%  regs {d.get('registers', 0):.0f}")
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
