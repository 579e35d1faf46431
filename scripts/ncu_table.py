"""Per-kernel table from an ncu --set full report: duration, DRAM bytes and throughput, L1/L2 utilisation."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "GB"), ("dram__bytes_write.sum", "GB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"), ("launch__registers_per_thread", ""),
        ("sm__cycles_elapsed.avg.per_second", "GHz")]
SCALE = {"msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9,
         "Tbyte": 1e3, "cycle/second": 1e-9, "cycle/nsecond": 1.0, "cycle/usecond": 1e-3}


def table(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k, _ in KEYS if k in hdr}
    ni = hdr.index("Kernel Name")
    lines = ["kernel | " + " | ".join(f"{k.split('.')[0].split('__')[1]} ({u})" for k, u in KEYS if k in idx)]
    for r in rows[2:]:
        vals = []
        for k, u in KEYS:
            if k not in idx:
                continue
            v = r[idx[k]].replace(",", "")
            try:
                x = float(v) * SCALE.get(units[idx[k]], 1.0)
                vals.append(f"{x:.3g}")
            except ValueError:
                vals.append(v)
        name = r[ni].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
        lines.append(name.split("(")[0][:40] + " | " + " | ".join(vals))
    return "\n".join(lines)


if __name__ == "__main__":
    print(table(sys.argv[1]))
