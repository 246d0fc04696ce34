"""Top SASS lines of an ncu capture by warp-stall samples (and the CUDA
source lines they map to): python scripts/ncu_hot.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
src = h.index("Source")
tot = sum(float(r[si] or 0) for r in data)
toti = sum(float(r[ii] or 0) for r in data)
print(f"total samples {tot:.0f}, warp instructions executed {toti:.0f}")
idx = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:N]
for i in sorted(idx):
    r = data[i]
    print(f"{i:5d} {float(r[si]):8.0f} {100*float(r[si])/tot:5.1f}%  inst {float(r[ii] or 0):12.0f}  {r[src].strip()[:90]}")
