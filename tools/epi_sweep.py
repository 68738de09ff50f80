"""A/B timings of the benched GEMM shapes under gemm.cu debug knobs (tpx_debug_gemm_mn_desc).

    python tools/epi_sweep.py [knobset ...]     knobset = "name=k:v,k:v" (or "base")
Each knob set is applied, the shapes are timed (tpx_gemm_timed, median of 5 x 20 launches),
then the knobs are reset to their defaults.  Development tool (not product, not a test)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04170_b200 import native  # noqa: E402
from tools.gemm_check import bench  # noqa: E402

DEFAULTS = {4: 0, 10: 1, 11: 0, 12: 1, 15: 0, 16: 4, 5: 1, 7: 0, 8: 0, 18: 0}
SHAPES = [("bwd_w+sgd tf32", (8192, 8192, 512, True, False), [3, 6], 0),
          ("bwd_w+sgd bf16", (8192, 8192, 512, True, False), [3, 6], 2),
          ("fwd+act tf32", (512, 8192, 8192, False, False), [1], 0),
          ("bwd_x+dact tf32", (512, 8192, 8192, False, True), [2], 0)]


def knob(k, v):
    native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(k), ctypes.c_uint(v))


def main():
    sets = sys.argv[1:] or ["base"]
    only = os.environ.get("SHAPES")
    for ks in sets:
        name, _, spec = ks.partition("=")
        pairs = [tuple(int(x) for x in kv.split(":")) for kv in spec.split(",") if kv]
        for k, v in pairs:
            knob(k, v)
        for label, shp, epi, prec in SHAPES:
            if only and not any(o in label for o in only.split(",")):
                continue
            r = [bench(*shp, iters=20, precision=prec, epi=epi) for _ in range(5)]
            ms = statistics.median(x[0] for x in r)
            gbs = statistics.median(x[2] for x in r)
            tf = statistics.median(x[1] for x in r)
            print(f"sweep {name:14s} {label:16s} {ms * 1e3:8.1f} us {tf:7.1f} TF/s {gbs:7.0f} GB/s", flush=True)
        for k, _ in pairs:
            knob(k, DEFAULTS.get(k, 0))


if __name__ == "__main__":
    main()
