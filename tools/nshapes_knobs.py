"""A/B of the small-M (weight-streaming) per-GPU GEMM shapes of cfg2 at N = 2 / 4 / 8 under gemm.cu
debug knobs: python tools/nshapes_knobs.py name=k:v,k:v ...  (development tool)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402
from tools.gemm_check import bench  # noqa: E402

SHAPES = [(m, 8192, 8192, False, tb, [2 if tb else 1]) for m in (64, 128, 256) for tb in (False, True)]
for ks in sys.argv[1:] or ["base"]:
    name, _, spec = ks.partition("=")
    pairs = [tuple(int(x) for x in kv.split(":")) for kv in spec.split(",") if kv]
    for k, v in pairs:
        native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(k), ctypes.c_uint(v))
    for M, N, K, ta, tb, epi in SHAPES:
        ms = statistics.median(bench(M, N, K, ta, tb, iters=20, epi=epi)[0] for _ in range(5))
        info = native.last_launch()
        print(f"{name:10s} M={M:4d} {'NT' if tb else 'NN'}: {ms * 1e3:6.1f} us  {256e6 / ms / 1e9:5.2f} TB/s(w)  "
              f"swap={info.get('swap')} pair={info.get('pair')} bn={info.get('bn')} sk={info.get('stream_k')} group={info.get('group')}", flush=True)
    for k, v in pairs:  # reset to defaults
        native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(k), ctypes.c_uint({29: 128, 30: 3, 23: 0, 6: 0, 9: 0}.get(k, 0)))
