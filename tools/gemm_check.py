"""GPU smoke + micro-benchmark of the tcgen05 GEMM through the C ABI (tpx_gemm).

    python tools/gemm_check.py [--bench]
Compares against torch fp64 matmul of the same fp32 inputs: normwise error
max|d| / max|ref| must be <= 2e-3 (TF32 inputs, fp32 accumulate).
"""
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_04170_b200 import native  # noqa: E402


def run(M, N, K, ta, tb, epi=None, pad=0, precision=0):
    dev = "cuda"
    dt = torch.bfloat16 if precision == 2 else torch.float32
    g = torch.Generator(device=dev).manual_seed(M * 7 + N * 3 + K)
    def padded(t):  # 16-byte row pitch (TMA), as the executor's buffers have
        al = 16 // t.element_size()
        cols = t.shape[1]
        if cols % al == 0 and not pad:
            return t
        return torch.nn.functional.pad(t, (0, (-cols) % al + pad))[:, :cols]

    A = padded((torch.rand((K, M) if ta else (M, K), device=dev, generator=g) * 2 - 1).to(dt))
    B = padded((torch.rand((N, K) if tb else (K, N), device=dev, generator=g) * 2 - 1).to(dt))
    C = padded(torch.full((M, N), float("nan"), device=dev, dtype=dt))
    outs = []
    if epi:
        for op in epi:
            outs.append(padded(torch.full((M, N), float("nan"), device=dev, dtype=dt)))
    W = padded((torch.rand((M, N), device=dev, generator=g) * 2 - 1).to(dt))
    native.gemm(A, B, ta, tb, C, epi=[(op, 0.01, W if op >= 4 else None, o) for op, o in zip(epi or [], outs)],
                precision=precision)
    torch.cuda.synchronize()
    ref = (A.double().T if ta else A.double()) @ (B.double().T if tb else B.double())
    err = ((C.double() - ref).abs().max() / ref.abs().max()).item()
    res = [err]
    prev = ref
    for op, o in zip(epi or [], outs):
        if precision == 2:
            prev = prev.to(torch.bfloat16).double()  # each stage reads the stored (bf16) value
        if op == 1:
            prev = torch.tanh(prev)
        elif op == 2:
            prev = 1 - torch.tanh(prev) ** 2
        elif op == 3:
            prev = 0.01 * prev
        elif op == 5:
            prev = prev - W.double()
        elif op == 6:
            prev = W.double() - prev
        # the epilogue carries the product's absolute error (tanh / 1-tanh^2 have gain <= 1):
        # normalise by the product's scale, like the product itself
        res.append(((o.double() - prev).abs().max() / max(prev.abs().max().item(), ref.abs().max().item(), 1e-30)).item())
    return res


def bench(M, N, K, ta, tb, iters=20, precision=0, epi=None):
    dt = torch.bfloat16 if precision == 2 else torch.float32
    A = torch.rand((K, M) if ta else (M, K), device="cuda").to(dt)
    B = torch.rand((N, K) if tb else (K, N), device="cuda").to(dt)
    C = torch.empty((M, N), device="cuda", dtype=dt)
    W = torch.rand((M, N), device="cuda").to(dt)
    outs = [torch.empty((M, N), device="cuda", dtype=dt) for _ in (epi or [])]
    e = [(op, 0.01, W if op >= 4 else None, o) for op, o in zip(epi or [], outs)]
    ms = native.gemm(A, B, ta, tb, C, epi=e, precision=precision, warmup=3, iters=iters)
    tf = 2 * M * N * K / ms / 1e9
    nb = (2 if precision == 2 else 4) * (M * K + K * N + M * N * (1 + len(epi or [])) + sum(M * N for op in (epi or []) if op >= 4))
    return ms, tf, nb / ms / 1e6


def diag():
    import ctypes
    L = native.lib()
    for lbo, sbo in [(4096, 512), (512, 4096), (4096, 1024), (1024, 4096)]:
        L.tpx_debug_gemm_mn_desc(ctypes.c_uint(lbo), ctypes.c_uint(sbo))
        for c in [(128, 128, 32, False, False), (128, 128, 8, False, False), (256, 256, 64, True, False)]:
            M, N, K, ta, tb = c
            A = torch.rand((K, M) if ta else (M, K), device="cuda") * 2 - 1
            B = torch.rand((N, K) if tb else (K, N), device="cuda") * 2 - 1
            C = torch.full((M, N), float("nan"), device="cuda")
            native.gemm(A, B, ta, tb, C)
            ref = (A.double().T if ta else A.double()) @ (B.double().T if tb else B.double())
            err = ((C.double() - ref).abs().max() / ref.abs().max()).item()
            print(f"lbo={lbo} sbo={sbo} case={c} err={err:.3g} nan={C.isnan().sum().item()} "
                  f"zeros={(C == 0).sum().item()} cmax={C.abs().max().item():.3g} refmax={ref.abs().max().item():.3g}")
            if K == 8 and lbo == 4096:
                r = ref.float()
                print("  C[0,:4]", C[0, :4].tolist(), " ref[0,:4]", r[0, :4].tolist())
    L.tpx_debug_gemm_mn_desc(ctypes.c_uint(0), ctypes.c_uint(0))


def main():
    if "--diag" in sys.argv:
        diag()
    for kv in filter(None, os.environ.get("TPX_GEMM_KNOBS", "").split(",")):
        k, v = kv.split(":")  # debug knobs of gemm.cu (tpx_debug_gemm_mn_desc)
        native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(int(k)), ctypes.c_uint(int(v)))
    if "--one" in sys.argv:
        # --one M N K ta tb [epi,...]: one timed configuration (for ncu)
        i = sys.argv.index("--one")
        M, N, K, ta, tb = (int(x) for x in sys.argv[i + 1:i + 6])
        epi = [int(x) for x in sys.argv[i + 6].split(",")] if len(sys.argv) > i + 6 and sys.argv[i + 6] != "-" else None
        prec = int(sys.argv[i + 7]) if len(sys.argv) > i + 7 else 0
        ms, tf, gb = bench(M, N, K, bool(ta), bool(tb), iters=3, epi=epi, precision=prec)
        print(f"one {(M, N, K, ta, tb)} epi={epi}: {ms:.3f} ms {tf:.1f} TFLOP/s {gb:.0f} GB/s")
        return
    cases = [
        (128, 128, 32, False, False), (128, 256, 64, False, True), (256, 256, 256, True, False),
        (512, 1024, 1024, False, False), (512, 1024, 1024, False, True), (1024, 1024, 512, True, False),
        (64, 1024, 1024, False, False), (64, 1024, 1024, False, True), (32, 2048, 4096, False, False),
        (4, 4096, 4096, False, False), (200, 300, 100, False, False), (1000, 136, 72, True, True),
        (64, 1000, 4096, False, False), (16, 1000, 1024, False, True),
    ]
    ok = True
    for c in cases:
        errs = run(*c)
        good = all(e <= 2e-3 for e in errs)
        ok &= good
        print(f"{'ok ' if good else 'BAD'} M,N,K,ta,tb={c} err={errs}")
    for epi in ([1, 2], [3, 6], [1]):
        errs = run(512, 512, 256, False, False, epi=epi)
        good = all(e <= 2e-3 for e in errs)
        ok &= good
        print(f"{'ok ' if good else 'BAD'} epilogue {epi} err={errs}")
    errs = run(32, 512, 512, False, False, epi=[3, 6])
    print(f"{'ok ' if all(e <= 2e-3 for e in errs) else 'BAD'} swapped epilogue err={errs}")
    # 3xTF32: fp32-accurate products
    for c in cases:
        errs = run(*c, precision=1)
        good = all(e <= 1e-5 for e in errs)
        ok &= good
        print(f"{'ok ' if good else 'BAD'} 3xTF32 M,N,K,ta,tb={c} err={errs}")
    errs = run(512, 512, 256, False, False, epi=[1, 2], precision=1)
    good = all(e <= 5e-6 for e in errs)
    ok &= good
    print(f"{'ok ' if good else 'BAD'} 3xTF32 epilogue [1,2] err={errs}")    # bf16 storage (kind::f16): products of bf16 operands in fp32, outputs rounded to bf16
    for c in cases:
        errs = run(*c, precision=2)
        good = all(e <= 8e-3 for e in errs)
        ok &= good
        print(f"{'ok ' if good else 'BAD'} bf16 M,N,K,ta,tb={c} err={errs}")
    for epi in ([1, 2], [3, 6]):
        for c in [(512, 512, 256, False, False), (256, 512, 512, True, False), (32, 512, 512, False, False)]:
            errs = run(*c, epi=epi, precision=2)
            good = all(e <= 8e-3 for e in errs)
            ok &= good
            print(f"{'ok ' if good else 'BAD'} bf16 epilogue {epi} {c} err={errs}")

    if "--bench" in sys.argv:
        L = native.lib()

        def med(c, epi=None, reps=5):
            r = sorted(bench(*c, epi=epi) for _ in range(reps))
            return r[len(r) // 2]

        for c, epi in [((512, 8192, 8192, False, False), [1]), ((512, 8192, 8192, False, True), [2]),
                       ((8192, 8192, 512, True, False), [3, 6]), ((8192, 8192, 512, True, False), None),
                       ((64, 8192, 8192, False, False), None), ((64, 8192, 8192, False, True), None),
                       ((64, 8192, 1024, True, False), [3, 6]),
                       ((4, 32768, 32768, False, False), None),
                       ((4096, 4096, 4096, False, False), None), ((8192, 8192, 8192, False, True), None)]:
            ms, tf, gb = med(c, epi)
            print(f"bench {c} epi={epi}: {ms:.3f} ms  {tf:.1f} TFLOP/s  {gb:.0f} GB/s(min bytes)")
        for c, epi in [((512, 8192, 8192, False, False), [1]), ((512, 8192, 8192, False, True), [2]),
                       ((8192, 8192, 512, True, False), [3, 6]), ((8192, 8192, 8192, False, True), None)]:
            ms, tf, gb = sorted(bench(*c, epi=epi, precision=2) for _ in range(5))[2]
            print(f"bench bf16 {c} epi={epi}: {ms:.3f} ms  {tf:.1f} TFLOP/s  {gb:.0f} GB/s(min bytes)")
        # interleaved A/B knob experiments: (knob, value) pairs, baseline (0-reset) between
        shapes = [((512, 8192, 8192, False, False), None), ((512, 8192, 8192, False, True), None),
                  ((8192, 8192, 512, True, False), [3, 6]), ((64, 8192, 8192, False, False), None),
                  ((4096, 4096, 4096, False, False), None), ((8192, 8192, 8192, False, True), None)]
        variants = [("base", []), ("nopair", [(6, 1)]), ("spin", [(5, 2)]), ("st4", [(4, 4)])]
        res = {}
        for rep in range(2):
            for name, knobs in variants:
                for k, v in knobs:
                    L.tpx_debug_gemm_mn_desc(ctypes.c_uint(k), ctypes.c_uint(v))
                for c, epi in shapes:
                    res.setdefault((name, c), []).append(bench(*c, epi=epi)[0])
                for k, v in knobs:
                    L.tpx_debug_gemm_mn_desc(ctypes.c_uint(k), ctypes.c_uint(0 if k != 2 else 0))
        for c, epi in shapes:
            print("knobs", c, epi, "  ".join(f"{n}={min(res[(n, c)]):.3f}" for n, _ in variants))
    print("ALL OK" if ok else "FAILURES")


if __name__ == "__main__":
    main()
