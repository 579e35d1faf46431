#!/usr/bin/env python
"""Stall-reason and traffic summary of one kernel in an ncu --set full report (read here, no GPU needed).
usage: python scripts/ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for v in rows[2:]:
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    print(d.get("Kernel Name", "?")[:80])
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
              "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"):
        if k in d:
            print(f"  {k:60s} {d[k]:>14s} {u.get(k, '')}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k] or 0) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1.0
    print("  stalls:", ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:7]))
