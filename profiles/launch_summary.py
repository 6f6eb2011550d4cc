"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into
per-kernel totals for one bench step.  Usage: launch_summary.py launches.csv [first_id last_id]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
mi = hdr.index("Metric Name") if "Metric Name" in hdr else None  # (lists with several metrics per launch)
ks = [(int(r[ii]), r[ki].split("(")[0].replace("void ", "").replace("mprkb::", "")[:70], float(r[vi].replace(",", "")))
      for r in rows[hdr_i + 1:] if len(r) > vi and (mi is None or r[mi] == "gpu__time_duration.sum")]
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    ks = [k for k in ks if lo <= k[0] <= hi]
tot = collections.OrderedDict()
for _, k, t in ks:
    c, s = tot.get(k, (0, 0.0))
    tot[k] = (c + 1, s + t)
all_ns = sum(s for _, s in tot.values())
print(f"{'kernel':72s} {'count':>5s} {'us':>9s} {'share':>6s}")
for k, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:72s} {c:5d} {s / 1e3:9.1f} {100 * s / all_ns:5.1f}%")
print(f"{'total':72s} {sum(c for c, _ in tot.values()):5d} {all_ns / 1e3:9.1f}")
