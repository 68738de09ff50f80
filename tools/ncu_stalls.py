"""Top stall sites of an .ncu-rep source page (SASS), e.g. python tools/ncu_stalls.py rep [n]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
tot = sum(int(r[si]) for r in data if r[si].isdigit())
print("total samples", tot)
idx = {r[0]: i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:n]:
    i = idx[r[0]]
    ctx = " | ".join(x[1].strip()[:50] for x in data[max(0, i - 2):i])
    print(f"{r[si]:>6} {r[0][-5:]} exec={r[ie]:>8}  {r[1].strip()[:70]:70s}  <= {ctx}")
