"""Median timings of a few GEMM configurations (layout x epilogue), for A/B decisions."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_check import bench  # noqa: E402

cfgs = [((8192, 8192, 512, True, False), [3, 6]), ((8192, 8192, 512, False, True), [3, 6]),
        ((8192, 8192, 512, True, False), None), ((8192, 8192, 512, False, True), None),
        ((8192, 8192, 512, False, True), [3]), ((8192, 8192, 512, False, True), [1])]
for c, e in cfgs:
    r = sorted(bench(*c, epi=e) for _ in range(7))[3]
    print(f"sweep {c} epi={e}: {r[0]:.3f} ms {r[1]:.1f} TFLOP/s {r[2]:.0f} GB/s")
