"""Summarise an ncu launch-list CSV (gpu__time_duration.sum, optionally dram bytes):
per-kernel launches, total / average time, share of GPU time, DRAM bytes and GB/s."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ni, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
ii = h.index("ID")
tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launch = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    name = re.sub(r"^void ", "", r[ki]).replace("<unnamed>::", "").split("(")[0]
    names[r[ii]] = name
    v = float(r[vi].replace(",", ""))
    if r[ni].startswith("gpu__time_duration"):
        launch[r[ii]]["us"] = v * tscale[r[ui]]
    elif r[ni].startswith("dram__bytes"):
        launch[r[ii]]["bytes"] = launch[r[ii]].get("bytes", 0.0) + v * bscale[r[ui]]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in launch.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("us", 0.0)
    a[2] += m.get("bytes", 0.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>11s} {'avg_us':>10s} {'share':>6s} {'dram_GB':>9s} {'GB/s':>7s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:40]:40s} {n:8d} {t:11.1f} {t / n:10.2f} {100 * t / tot:5.1f}% {b / 1e9:9.3f} {b / (t * 1e3) if t else 0:7.0f}")
print(f"{'TOTAL':40s} {sum(v[0] for v in agg.values()):8d} {tot:11.1f}")
