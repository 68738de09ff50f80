"""Print the kernel variant (tpx_gemm_last_launch) the GEMM picks for given shapes:
    python tools/launch_info.py M,N,K,ta,tb[,epi:epi] ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402

for arg in sys.argv[1:]:
    parts = arg.split(",")
    M, N, K, ta, tb = (int(x) for x in parts[:5])
    epi = [int(x) for x in parts[5].split(":")] if len(parts) > 5 else []
    A = torch.rand((K, M) if ta else (M, K), device="cuda")
    B = torch.rand((N, K) if tb else (K, N), device="cuda")
    C = torch.empty(M, N, device="cuda")
    W = torch.rand(M, N, device="cuda")
    outs = [torch.empty(M, N, device="cuda") for _ in epi]
    ms = native.gemm(A, B, bool(ta), bool(tb), C, epi=[(op, 0.01, W if op >= 4 else None, o) for op, o in zip(epi, outs)],
                     warmup=2, iters=10)
    print((M, N, K, ta, tb, epi), f"{ms * 1e3:.1f} us", native.last_launch(), flush=True)
