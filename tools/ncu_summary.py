"""Summarise ncu output for profiles/: a launch list CSV (gpu__time_duration.sum) and/or an
.ncu-rep (--set full) into a short text report (per-kernel time share; per-launch DRAM bytes,
tensor-pipe %, DRAM %, L2 %, registers)."""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1 if d["Metric Unit"] == "us" else 1e3)
                out.append((d["Kernel Name"].split("(")[0].replace("void ", ""), d["Grid Size"], v))
    return out


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
    out = []
    for r in rows[2:]:
        out.append({w: (r[hdr.index(w)] + " " + units[hdr.index(w)]).strip() for w in want if w in hdr})
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        if p.endswith(".csv"):
            L = launches(p)
            tot = collections.defaultdict(lambda: [0, 0.0])
            for name, grid, us in L:
                tot[(name, grid)][0] += 1
                tot[(name, grid)][1] += us
            s = sum(v[1] for v in tot.values())
            print(f"# launch list {p}: {len(L)} launches, {s:.1f} us total (ncu-serialised, cold-cache)")
            for (name, grid), (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
                print(f"{us / s * 100:6.2f}%  {n:4d} x {us / n:9.2f} us  grid {grid:14s} {name}")
        else:
            for d in full(p):
                print("---")
                for k, v in d.items():
                    print(f"  {k}: {v}")
