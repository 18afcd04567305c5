"""Dev tool: per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_summary.py launches.csv [steps]"""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in csv.reader(open(path)):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        agg[d["Kernel Name"][:90]][0] += 1
        agg[d["Kernel Name"][:90]][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.3f} ms over {steps} step(s): {tot / steps:.3f} ms per step (cold-cache, serialised)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1] / steps:9.3f} ms/step {v[0]:5d} launches {100 * v[1] / tot:5.1f}%  {k}")
