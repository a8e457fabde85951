"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        k = r["Kernel Name"][:60]
        v = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Unit", "ns") == "usecond":
            v *= 1e3
        agg[k][0] += 1
        agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'total us':>10s} {'us/launch':>10s} share")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {v[0]:5d} {v[1] / 1e3:10.1f} {v[1] / max(v[0], 1) / 1e3:10.2f} {v[1] / tot:.3f}")
