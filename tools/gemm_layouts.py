"""Operand-majorness sweep of the tcgen05 GEMM on one shape (median of 5 x 20 runs).

    python tools/gemm_layouts.py M N K [precision: 0 tf32, 2 bf16] [epi,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_check import bench  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 0
epi = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else None
for ta in (False, True):
    for tb in (False, True):
        r = sorted(bench(M, N, K, ta, tb, precision=prec, epi=epi) for _ in range(5))[2]
        print(f"layout prec={prec} ta={int(ta)} tb={int(tb)} {M}x{N}x{K} epi={epi}: {r[0]:.3f} ms {r[1]:.1f} TFLOP/s {r[2]:.0f} GB/s")
