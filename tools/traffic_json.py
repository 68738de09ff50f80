"""profiles/traffic.json from an ncu --set full capture of one step's GEMMs (tools/ncu_step.py):
DRAM bytes (read + write) per launch, averaged per GEMM class in launch order fwd/bwd_w/bwd_x."""
import csv
import json
import subprocess
import sys

rep, order = sys.argv[1], sys.argv[2].split(",")  # order: class name of each captured launch
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
h = rows[0]
ir, iw, it = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = {}
for cls, row in zip(order, rows[2:]):
    b = float(row[ir]) * unit[rows[1][ir]] + float(row[iw]) * unit[rows[1][iw]]
    acc.setdefault(cls, []).append(b)
src = (f"{rep} (ncu --set full --clock-control none -k regex:gemm, one cfg2 k=0 step, tools/ncu_step.py): "
       "dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged per class")
out = {c: {"dram_bytes_per_launch": sum(v) / len(v), "source": src} for c, v in acc.items()}  # bench.py reads this
json.dump(out, sys.stdout, indent=1)
