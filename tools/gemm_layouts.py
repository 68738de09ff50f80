"""Operand-majorness sweep of the tcgen05 GEMM on one shape (median of 5 x 20 runs)."""
import sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from tools.gemm_check import bench  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 8192, 512)
for ta in (False, True):
    for tb in (False, True):
        r = sorted(bench(M, N, K, ta, tb) for _ in range(5))[2]
        print(f"layout ta={int(ta)} tb={int(tb)} {M}x{N}x{K}: {r[0]:.3f} ms {r[1]:.1f} TFLOP/s")
