"""Per-kernel totals and shares from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).
usage: python tools/launch_shares.py X.csv [top]"""
import collections
import csv
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 10
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "second": 1e3, "s": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    a = agg[r["Kernel Name"][:100]]
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"| kernel | launches | total ms | mean ms | share |\n|---|---:|---:|---:|---:|")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"| `{k}` | {a[0]} | {a[1]:.2f} | {a[1] / a[0]:.3f} | {100 * a[1] / tot:.1f}% |")
