"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
agg = defaultdict(lambda: [0.0, 0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v = v / 1e3 if unit == "ns" else v * 1e3 if unit == "msecond" else v if unit in ("us", "usecond") else v
    agg[name][0] += v
    agg[name][1] += 1
tot = sum(a[0] for a in agg.values())
print(f"total {tot:.1f} us over {sum(a[1] for a in agg.values())} launches")
for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{us:10.1f} us {100 * us / tot:5.1f}% {n:5d}x {us / n:8.2f} us/launch  {k}")
