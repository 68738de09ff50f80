"""Kernel-level GPU tests through the C ABI (tpx_gemm): the tcgen05 tile GEMM for every
transpose form the plans use (NN fwd, TN bwd_w, NT bwd_x — graph.cpp:192-209), edge tiles,
tiny M (replicated-weight tiles), split-K, strided views, and fused epilogues, against a torch
fp64 reference of the same fp32 inputs (normwise max|d| / max|ref|):
    TF32  <= 2e-3      3xTF32 (PREC_FP32) <= 1e-5
"""
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # M, N, K, ta, tb
    (128, 128, 32, False, False), (128, 256, 64, False, True), (256, 256, 256, True, False),
    (512, 1024, 1024, False, False), (512, 1024, 1024, False, True), (1024, 1024, 512, True, False),
    (64, 1024, 1024, False, False), (64, 1024, 1024, False, True), (32, 2048, 4096, False, False),
    (4, 4096, 4096, False, False), (200, 300, 100, False, False), (1000, 136, 72, True, True),
    (64, 1000, 4096, False, False), (16, 1000, 1024, False, True), (8, 8, 8, False, False),
    (1, 64, 64, False, False), (512, 8192, 1024, False, False),
]


def _run(M, N, K, ta, tb, precision, epi=None):
    import torch
    from paper_1805_04170_b200 import native
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(M * 7 + N * 3 + K)
    A = torch.rand((K, M) if ta else (M, K), device=dev, generator=g) * 2 - 1
    B = torch.rand((N, K) if tb else (K, N), device=dev, generator=g) * 2 - 1
    C = torch.full((M, N), float("nan"), device=dev)
    W = torch.rand((M, N), device=dev, generator=g) * 2 - 1
    outs = [torch.full((M, N), float("nan"), device=dev) for _ in (epi or [])]
    native.gemm(A, B, ta, tb, C, epi=[(op, 0.01, W if op >= 4 else None, o) for op, o in zip(epi or [], outs)],
                precision=precision)
    torch.cuda.synchronize()
    ref = (A.double().T if ta else A.double()) @ (B.double().T if tb else B.double())
    return C, ref, W, outs


def _nw(got, ref):
    return ((got.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s[:3])) + ("T" if s[3] else "N") + ("T" if s[4] else "N"))
@pytest.mark.parametrize("precision", [0, 1], ids=["tf32", "fp32"])
def test_gemm(shape, precision):
    C, ref, _, _ = _run(*shape, precision)
    assert _nw(C, ref) <= (2e-3 if precision == 0 else 1e-5)


@pytest.mark.parametrize("precision", [0, 1], ids=["tf32", "fp32"])
def test_gemm_update_epilogue(precision):
    """bwd_w -> step (scale by lr) -> upd (w - wd): the fused SGD update (gemm.h EPI_SCALE,
    EPI_SUB_OP), each intermediate stored."""
    import torch
    C, ref, W, (wd, wn) = _run(512, 1024, 256, True, False, precision, epi=[3, 6])
    tol = 2e-3 if precision == 0 else 1e-5
    assert _nw(C, ref) <= tol
    assert _nw(wd, 0.01 * ref) <= tol
    assert ((wn.double() - (W.double() - 0.01 * ref)).abs().max() / (0.01 * ref).abs().max()).item() <= tol
    assert torch.equal(wd, 0.01 * C)


def test_gemm_act_epilogue_bitexact():
    """fwd -> act (tanh) fused: the stored activation is tanhf of the stored product."""
    import torch
    C, ref, _, (h,) = _run(256, 512, 128, False, False, 1, epi=[1])
    assert torch.equal(h, torch.tanh(C)) or (h - torch.tanh(C)).abs().max().item() <= 2e-7


@pytest.mark.parametrize("shape,epi", [((1024, 4096, 256, True, False), [3, 6]), ((512, 1024, 1024, False, True), [1]),
                                       ((64, 1024, 1024, False, False), None), ((1000, 136, 72, True, True), None)],
                         ids=["tn_update", "nt_act", "small", "edge"])  # (pair kernels: test_gpu_fullsize.py)
def test_gemm_dynamic_schedule(shape, epi):
    """Whole-tile schedules handed out by the device tile counter (debug knob (10, 0)):
    same results as the static per-CTA lists, twice in a row (the counter re-arms itself)."""
    import torch
    from paper_1805_04170_b200 import native
    base = _run(*shape, 0, epi=epi)
    native.lib().tpx_debug_gemm_mn_desc(10, 0)
    try:
        for _ in range(2):
            got = _run(*shape, 0, epi=epi)
            assert torch.equal(got[0], base[0])
            for a, b in zip(got[3], base[3]):
                assert torch.equal(a, b)
    finally:
        native.lib().tpx_debug_gemm_mn_desc(10, 1)


# MN-major (transposed) TF32 operands: the k-group-major stage (4-D TMA map) when the MN extent
# is a multiple of 32 and K a multiple of 4, else the chunk-major stage (3-D / 2-D maps).
MN_SHAPES = [  # M, N, K, ta, tb
    (256, 256, 4, True, False), (256, 512, 12, True, False), (384, 256, 36, True, False),
    (512, 256, 100, True, True), (96, 640, 64, True, False), (256, 96, 64, False, False),
    (256, 256, 30, True, False), (80, 256, 64, True, False), (256, 200, 64, False, False),
    (2048, 2048, 512, True, False), (512, 2048, 2048, False, False),
]


@pytest.mark.parametrize("shape", MN_SHAPES, ids=lambda s: "x".join(map(str, s[:3])) + ("T" if s[3] else "N") + ("T" if s[4] else "N"))
@pytest.mark.parametrize("precision", [0, 1], ids=["tf32", "fp32"])
def test_mn_major_stage_layouts(shape, precision):
    """Both MN-major stage layouts against torch fp64, and bit-identical to each other (the same
    products in the same k order; only the shared-memory arrangement differs)."""
    import ctypes

    import torch
    from paper_1805_04170_b200 import native
    C, ref, _, _ = _run(*shape, precision)
    assert _nw(C, ref) <= (2e-3 if precision == 0 else 1e-5)
    native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(25), ctypes.c_uint(0))  # chunk-major stages
    try:
        C0, _, _, _ = _run(*shape, precision)
    finally:
        native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(25), ctypes.c_uint(1))
    assert torch.equal(C, C0)


def test_weight_streaming_tile_width():
    """A single row of P tiles against a wide weight (the cfg2 per-GPU fwd shape at N = 4) takes
    128-wide tiles (<= 3 stream-K cuts each, gemm.cu g_max_cuts) and stays exact."""
    from paper_1805_04170_b200 import native
    C, ref, _, _ = _run(128, 8192, 8192, False, False, 0)
    info = native.last_launch()
    assert (info["bn"], info["pair"], info["swap"], info["stream_k"]) == (128, 0, 0, 1)
    assert _nw(C, ref) <= 2e-3
