"""Feasibility probe: do bwd_w + SGD (HBM/L2-bound) and bwd_x (tensor-bound) overlap when each
runs on part of the SMs on its own stream?  Times each alone at several SM caps, then both at
once (two host threads, two streams).  Development tool."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402

dev = "cuda"
x = torch.rand(512, 8192, device=dev)
g = torch.rand(512, 8192, device=dev)
w = torch.rand(8192, 8192, device=dev)
gw, wd, wn = (torch.empty(8192, 8192, device=dev) for _ in range(3))
h = torch.empty(512, 8192, device=dev)
d = torch.empty(512, 8192, device=dev)


def bwd_w(iters, stream):
    return native.gemm(x, g, True, False, gw, epi=[(3, 0.01, None, wd), (6, 0.01, w, wn)], stream=stream,
                       warmup=2, iters=iters)


def bwd_x(iters, stream):
    return native.gemm(g, w, False, True, h, epi=[(2, 0.0, None, d)], stream=stream, warmup=2, iters=iters)


for sms in ("148", "112", "96", "74", "52"):
    os.environ["TPX_GEMM_SMS"] = sms
    print(f"alone sms={sms}: bwd_w {bwd_w(20, None) * 1e3:.1f} us  bwd_x {bwd_x(20, None) * 1e3:.1f} us", flush=True)

for a, b in (("74", "74"), ("96", "52"), ("112", "36")):
    res = {}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(name, fn, sms, st):
        res[name] = fn(40, st.cuda_stream)

    os.environ["TPX_GEMM_SMS"] = a
    t1 = threading.Thread(target=run, args=("w", bwd_w, a, s1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t1.start()
    time.sleep(0.02)
    os.environ["TPX_GEMM_SMS"] = b
    t2 = threading.Thread(target=run, args=("x", bwd_x, b, s2))
    t2.start()
    t1.join()
    t2.join()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"concurrent bwd_w@{a} + bwd_x@{b}: per-iter bwd_w {res['w'] * 1e3:.1f} us, bwd_x {res['x'] * 1e3:.1f} us "
          f"(wall {wall * 1e3:.1f} ms for 40+40 incl. prepare)", flush=True)
