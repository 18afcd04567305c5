"""Dev: top CUDA source lines of an ncu report by warp-stall samples and by instructions executed
(ncu -i <rep> --page source --csv --print-source cuda,sass; needs -lineinfo).
usage: python tools/ncu_top.py report.ncu-rep [N]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, data = "?", []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 8 or r[2] != "-":
        continue
    try:
        data.append((float(r[4] or 0), float(r[7] or 0), f"{fname}:{r[0]}", r[1].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"total stall samples {tot:.0f}, warp instructions {toti:.4e}")
print("-- by stall samples")
for s, i, a, t in sorted(data, reverse=True)[:N]:
    print(f"{100 * s / tot:5.2f}% {100 * i / toti:5.2f}%i  {a:>20} {t[:100]}")
print("-- by instructions")
for s, i, a, t in sorted(data, key=lambda d: -d[1])[:N // 2]:
    print(f"{100 * s / tot:5.2f}% {100 * i / toti:5.2f}%i  {a:>20} {t[:100]}")
