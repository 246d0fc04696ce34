"""Warp-stall samples of an ncu capture aggregated by CUDA source line (needs
-lineinfo and --import-source on): python scripts/ncu_lines.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
src = h.index("Source")
ln = h.index("#") if "#" in h else 0
tot = sum(float(r[si] or 0) for r in data)
toti = sum(float(r[ii] or 0) for r in data)
print(f"total samples {tot:.0f}, warp instructions executed {toti:.0f}")
idx = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:N]
for i in sorted(idx):
    r = data[i]
    print(f"{r[ln]:>6} {float(r[si] or 0):8.0f} {100*float(r[si] or 0)/tot:5.1f}%  inst {float(r[ii] or 0):12.0f}  {r[src].strip()[:100]}")
