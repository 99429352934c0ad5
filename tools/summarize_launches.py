"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per kernel totals and shares)."""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ui, vi = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    name = re.sub(r"^void ", "", r[ki]).replace("<unnamed>::", "")
    name = name.split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':34s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:34s} {n:8d} {t:10.1f} {t / n:9.2f} {100 * t / tot:5.1f}%")
print(f"{'TOTAL':34s} {sum(v[0] for v in agg.values()):8d} {tot:10.1f}")
