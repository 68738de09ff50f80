"""Per-CTA timeline of one GEMM launch (debug knob (22, 1), tpx_debug_gemm_trace): where a
launch's fixed cost goes.  python tools/gemm_trace.py M,N,K,ta,tb[,epi:epi] ...
Milestones (us after the first CTA's entry): setup done, first TMA issued, first k-block landed,
MMA done, first accumulator ready, epilogue done, exit -- median and max over the active CTAs."""
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402

NAMES = ["entry", "setup", "tma0", "kb0", "mma_done", "acc0", "epi_done", "exit"]
L = native.lib()
for arg in sys.argv[1:]:
    parts = arg.split(",")
    M, N, K, ta, tb = (int(x) for x in parts[:5])
    epi = [int(x) for x in parts[5].split(":")] if len(parts) > 5 else []
    prec = int(os.environ.get("PREC", "0"))  # 2: bf16 storage
    dt = torch.bfloat16 if prec == 2 else torch.float32
    A = torch.rand((K, M) if ta else (M, K), device="cuda").to(dt)
    B = torch.rand((N, K) if tb else (K, N), device="cuda").to(dt)
    C = torch.empty(M, N, device="cuda", dtype=dt)
    W = torch.rand(M, N, device="cuda").to(dt)
    outs = [torch.empty(M, N, device="cuda", dtype=dt) for _ in epi]
    e = [(op, 0.01, W if op >= 4 else None, o) for op, o in zip(epi, outs)]
    native.gemm(A, B, bool(ta), bool(tb), C, epi=e, warmup=3, iters=5, precision=prec)
    L.tpx_debug_gemm_mn_desc(ctypes.c_uint(22), ctypes.c_uint(1))
    buf = (ctypes.c_uint64 * (320 * 8))()
    for i in range(320 * 8):
        buf[i] = 0
    native.gemm(A, B, bool(ta), bool(tb), C, epi=e, precision=prec)
    torch.cuda.synchronize()
    L.tpx_debug_gemm_trace(buf, 320 * 8)
    L.tpx_debug_gemm_mn_desc(ctypes.c_uint(22), ctypes.c_uint(0))
    info = native.last_launch()
    rows = [[buf[c * 8 + i] for i in range(8)] for c in range(info["units"] if info["units"] <= 320 else 320)]
    rows = [r for r in rows if r[0] and r[7]]
    t0 = min(r[0] for r in rows)
    print(f"{(M, N, K, ta, tb, epi)} units={info['units']} pair={info['pair']} bn={info['bn']} stream_k={info['stream_k']}")
    for i, nm in enumerate(NAMES):
        v = [(r[i] - t0) / 1e3 for r in rows if r[i]]
        if v:
            print(f"   {nm:9s} median {statistics.median(v):7.2f} us  max {max(v):7.2f} us  ({len(v)} CTAs)")
