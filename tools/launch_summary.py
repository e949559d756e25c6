"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list.
Usage: python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import sys

agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(d["Metric Unit"], 1.0)
    k = d["Kernel Name"][:100]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v[1] / tot * 100:5.1f}% {v[0]:5d} {v[1] / v[0] / 1e3:9.1f}us {k}")
