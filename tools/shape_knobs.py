"""A/B of arbitrary GEMM shapes under gemm.cu debug knobs (development tool):
    python tools/shape_knobs.py "M,N,K,ta,tb[,epi:epi]" ... -- name=k:v,k:v ...
Each knob set is applied, every shape is timed (median of 5 x 20 launches), then the knobs are
reset (DEFAULTS)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402
from tools.gemm_check import bench  # noqa: E402

DEFAULTS = {4: 0, 6: 0, 9: 0, 10: 1, 11: 0, 12: 1, 15: 0, 16: 4, 18: 0, 23: 0, 29: 128, 30: 3}
i = sys.argv.index("--")
shapes = []
for a in sys.argv[1:i]:
    p = a.split(",")
    shapes.append((tuple(int(x) for x in p[:5]), [int(x) for x in p[5].split(":")] if len(p) > 5 else None))
for ks in sys.argv[i + 1:] or ["base"]:
    name, _, spec = ks.partition("=")
    pairs = [tuple(int(x) for x in kv.split(":")) for kv in spec.split(",") if kv]
    for k, v in pairs:
        native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(k), ctypes.c_uint(v))
    for (M, N, K, ta, tb), epi in shapes:
        prec = int(os.environ.get("PREC", "0"))  # 2: bf16 storage
        ms = statistics.median(bench(M, N, K, bool(ta), bool(tb), iters=20, epi=epi, precision=prec)[0] for _ in range(5))
        info = native.last_launch()
        print(f"{name:10s} {(M, N, K, ta, tb)} epi={epi}: {ms * 1e3:7.1f} us  pair={info.get('pair')} bn={info.get('bn')} "
              f"sk={info.get('stream_k')} group={info.get('group')} stages={info.get('stages')}", flush=True)
    for k, v in pairs:
        native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(k), ctypes.c_uint(DEFAULTS.get(k, 0)))
