"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file X.csv`) per kernel name.
usage: python tools/launch_summary.py X.csv "<command line that produced it>" [per_step_kernel_regex]
Prints total / share / count / mean per kernel, then the kernels launched once per training step (those whose
count equals the step kernel's) with their share of one step."""
import csv
import re
import sys
from collections import OrderedDict


def main():
    path, cmd = sys.argv[1], sys.argv[2]
    step_re = re.compile(sys.argv[3] if len(sys.argv) > 3 else r"step_kernel")
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1.0, "nsecond": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1.0)
        rows.append((r["Kernel Name"], v))
    agg = OrderedDict()
    for name, v in rows:
        t = agg.setdefault(name, [0.0, 0])
        t[0] += v
        t[1] += 1
    total = sum(t[0] for t in agg.values())
    print(f"launch list: {cmd}")
    print("(cold-cache, serialised launches: compare shares, not absolute times). unit: ns\n")
    for name, (tot, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{tot / 1e6:10.3f} ms total {100 * tot / total:5.1f}%  n={n:3d}  mean {tot / n / 1e6:9.4f} ms  {name[:110]}")
    nstep = max((n for name, (_, n) in agg.items() if step_re.search(name)), default=0)
    per = [(name, tot / n) for name, (tot, n) in agg.items() if n == nstep and nstep > 0]
    step_ms = sum(m for _, m in per)
    print("\nper-step kernels (mean per launch) and their share of one training step:")
    for name, m in sorted(per, key=lambda kv: -kv[1]):
        print(f"{m / 1e6:10.4f} ms {100 * m / step_ms:6.1f}%  {name[:100]}")


if __name__ == "__main__":
    main()
