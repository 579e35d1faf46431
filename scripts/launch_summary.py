"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time per kernel name and share."""
import collections
import csv
import re
import sys


def summary(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        raw = re.sub(r"^void\s+", "", r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", ""))
        m = re.match(r"([A-Za-z_:][A-Za-z0-9_:]*)", raw)
        name = (m.group(1) if m else raw[:40]).split("::")[-1]
        t = re.match(r"[A-Za-z_:][A-Za-z0-9_:]*(<[^()]*?>)\(", raw)   # template arguments of our kernels
        if t and len(t.group(1)) < 24:
            name += t.group(1)
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"{'kernel':45s} {'launches':>8s} {'ms':>10s} {'share':>7s}"]
    for k, v in tot.most_common(top):
        out.append(f"{k:45s} {cnt[k]:8d} {v:10.3f} {100 * v / T:6.1f}%")
    out.append(f"{'total':45s} {sum(cnt.values()):8d} {T:10.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25))
