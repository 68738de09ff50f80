"""Per-GPU GEMM shapes of the cfg2 optimum at N = 2 / 4 / 8 (one logical device per GPU), each
timed alone on one B200: the compute part of the N-GPU step, with its roofline (max of FLOPs at
the TF32 peak and algorithmic bytes at the HBM peak).  Development / evidence tool."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_check import bench  # noqa: E402

peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
TC, HBM = peaks["bf16_tflops"] / 2 * 1e12, peaks["hbm_gbs"] * 1e9
rows = []
for n, m in ((1, 512), (2, 256), (4, 128), (8, 64)):
    shapes = [("fwd+act", (m, 8192, 8192, False, False), [1]), ("bwd_x+dact", (m, 8192, 8192, False, True), [2]),
              ("bwd_w+sgd", (8192 // n, 8192, 512, True, False), [3, 6])]
    tot = roof = 0.0
    for label, shp, epi in shapes:
        r = [bench(*shp, iters=20, epi=epi) for _ in range(5)]
        ms = statistics.median(x[0] for x in r)
        M, N, K = shp[:3]
        fl = 2.0 * M * N * K
        by = 4.0 * (M * K + K * N + M * N * (1 + len(epi)) + (M * N if 6 in epi else 0))
        rf = max(fl / TC, by / HBM) * 1e3
        tot += 5 * ms
        roof += 5 * rf
        print(f"N={n} {label:11s} {shp}: {ms * 1e3:7.1f} us  roofline {rf * 1e3:6.1f} us  frac {rf / ms:.2f}", flush=True)
        rows.append({"n": n, "what": label, "shape": shp[:3], "us": ms * 1e3, "roofline_us": rf * 1e3})
    print(f"N={n}: 15 GEMMs {tot:.3f} ms (roofline {roof:.3f} ms) -> compute-only {512 / (tot / 1e3):.0f} samples/s per job", flush=True)
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "nshapes.json")
json.dump(rows, open(out, "w"), indent=1)
