"""GPU numerics probe of the tcgen05 GEMM on structured (reference-like) operands: saturated
activations (exactly +-1) times sparse positive gradients (1 - tanh^2 of wide values), the data
the teacher-forced full-size tests feed bwd_w.  Compares every kernel variant (pair / single
CTA / 2-D boxes / no loader warp) with fp64 and with emulated operand roundings (tf32
truncation, tf32 round-to-nearest) on the same operands.

    python tools/numerics_probe.py [M N K]   (writes gpurun_out/numerics_probe.json)
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_04170_b200 import native  # noqa: E402


def nw(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max()).item()


def tf32_trunc(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


def tf32_rna(x):
    return ((x.view(torch.int32) + 0x1000) & ~0x1FFF).view(torch.float32)


def main():
    M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 8192, 512)
    g = torch.Generator(device="cuda").manual_seed(1)
    out = {}
    datasets = {
        "random": (torch.rand((K, M), device="cuda", generator=g) * 2 - 1,
                   torch.rand((K, N), device="cuda", generator=g) * 2 - 1),
        "saturated_x_sparse_g": (torch.sign(torch.randn((K, M), device="cuda", generator=g)),
                                 1 - torch.tanh(30 * torch.randn((K, N), device="cuda", generator=g)) ** 2),
        "x_sparse_g_dense": (torch.tanh(30 * torch.randn((K, M), device="cuda", generator=g)),
                             torch.rand((K, N), device="cuda", generator=g)),
    }
    knobs = {"default": [], "single_cta": [(6, 1)], "2d_boxes": [(3, 1)], "no_loader": [(12, 0)],
             "no_stream_hints": [(8, 1)], "3xtf32": [], "3xtf32_unbounded": [(13, 0)]}
    reset = {6: 0, 3: 0, 12: 1, 8: 0, 13: 16}
    for dname, (A, B) in datasets.items():
        A, B = A.float().contiguous(), B.float().contiguous()
        ref = A.double().t() @ B.double()
        fl_tr = tf32_trunc(A).double().t() @ tf32_trunc(B).double()
        fl_rn = tf32_rna(A).double().t() @ tf32_rna(B).double()
        row = {"floor_trunc": nw(fl_tr, ref), "floor_rna": nw(fl_rn, ref)}
        W = torch.rand((M, N), device="cuda", generator=g) * 2 - 1
        for kname, ks in knobs.items():
            for epi in (0, 1):
                for a, b in ks:
                    native.lib().tpx_debug_gemm_mn_desc(a, b)
                try:
                    C = torch.empty((M, N), device="cuda")
                    wd, wn = torch.empty_like(C), torch.empty_like(C)
                    e = [(3, 0.01, None, wd), (6, 0.0, W, wn)] if epi else None
                    native.gemm(A, B, True, False, C, epi=e, precision=1 if kname.startswith("3x") else 0)
                    torch.cuda.synchronize()
                    info = native.last_launch()
                    row[f"{kname}{'+sgd' if epi else ''}"] = {
                        "vs_fp64": nw(C, ref), "vs_floor_trunc": nw(C, fl_tr), "vs_floor_rna": nw(C, fl_rn),
                        "pair": info["pair"], "bn": info["bn"], "oloader": info["oloader"]}
                finally:
                    for a, _ in ks:
                        native.lib().tpx_debug_gemm_mn_desc(a, reset[a])
        out[dname] = row
        print(dname, json.dumps(row, indent=1), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"numerics_probe_{M}x{N}x{K}.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
