"""ncu probe of the executor's GEMM on the cfg2 shapes (not product): one launch per shape, plain
(no epilogue), next to tools/cublas_probe.py's cuBLAS launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402

prec = 2 if "bf16" in sys.argv else 0
dt = torch.bfloat16 if prec == 2 else torch.float32
for (M, N, K, ta, tb) in [(512, 8192, 8192, False, False), (512, 8192, 8192, False, True),
                          (8192, 8192, 512, True, False)]:
    A = torch.rand((K, M) if ta else (M, K), device="cuda").to(dt)
    B = torch.rand((N, K) if tb else (K, N), device="cuda").to(dt)
    C = torch.empty((M, N), device="cuda", dtype=dt)
    native.gemm(A, B, ta, tb, C, precision=prec, warmup=0, iters=1)
    torch.cuda.synchronize()
