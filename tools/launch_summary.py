"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares of device time, for profiles/:
python tools/launch_summary.py launches.csv "header line" > summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    tot[r[ki]] += v
    cnt[r[ki]] += 1
s = sum(tot.values())
print("unit: ns; " + (sys.argv[2] if len(sys.argv) > 2 else ""))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:90]:90s} launches={cnt[k]:4d} total={v:14.1f} share={100 * v / s:5.1f}%")
