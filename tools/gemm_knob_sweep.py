"""Time GEMM shapes under gemm.cu debug knobs: python tools/gemm_knob_sweep.py "M,N,K,ta,tb[,epi]" ... -- knob:value ..."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402
from tools.gemm_check import bench  # noqa: E402

args = sys.argv[1:]
cut = args.index("--") if "--" in args else len(args)
shapes, knobs = args[:cut], ["base"] + args[cut + 1:]
L = native.lib()
for sh in shapes:
    f = sh.split(",")
    M, N, K, ta, tb = (int(x) for x in f[:5])
    epi = [int(x) for x in f[5].split("+")] if len(f) > 5 else None
    prec = int(f[6]) if len(f) > 6 else 0
    for kn in knobs:
        if kn != "base":
            k, v = kn.split(":")
            L.tpx_debug_gemm_mn_desc(ctypes.c_uint(int(k)), ctypes.c_uint(int(v)))
        r = sorted(bench(M, N, K, bool(ta), bool(tb), epi=epi, precision=prec) for _ in range(5))[2]
        print(f"sweep {sh} knob={kn}: {r[0] * 1e3:.1f} us {r[1]:.1f} TFLOP/s {r[2]:.0f} GB/s")
        if kn != "base":
            L.tpx_debug_gemm_mn_desc(ctypes.c_uint(int(k)), ctypes.c_uint(0))
