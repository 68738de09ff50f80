"""GPU parity at the BENCHED sizes and for the BENCHED kernel variants (SURVEY §8(c) parity plan
items 2-4; round-1 verdict "next" #1).

Three layers of checks, all through the C ABI:

1. Kernel variants at the benched GEMM shapes (tpx_gemm + tpx_gemm_last_launch): the exact
   lowered shapes of cfg2 (gen_mlp(512, [8192]*6)) — fwd NN 512x8192x8192 + tanh (+ 1-tanh^2
   for the last layer), bwd_x NT 512x8192x8192 + 1-tanh^2, bwd_w TN 8192x8192x512 + SGD step
   and update — and the AlexNet-style conv grad_input GEMM TN 3456x100352x256, in TF32 and
   bf16.  Each test asserts the variant it covers (CTA pair, tile width, operand-loader warp),
   so a change in tile selection cannot silently drop coverage.  The product is compared with
   torch fp64 on the same stored operands; every fused stage with that stage applied in fp64
   (fp32: bit-exact for scale/sub) to the value the previous stage stored.
2. Whole plans at full size, per op, teacher-forced: the torch fp64 restatement of the
   reference's executor (oracle/torch_oracle.py, pinned to the reference's goldens by
   tests/test_torch_oracle.py) supplies every node's value; each op's input holders receive
   the oracle's values, only that op's lowered steps run, and its output holders are compared
   (normwise max|d|/max|ref| per block).  Ops fused into a producer's epilogue are checked
   against the op applied in fp64 to the values the fused launch stored.
3. Whole plans at full size, chained from seeded inputs, fp32-accurate path (3xTF32): gated at
   2x the MEASURED fp32 floor — the same graph run in plain fp32 by torch (no TF32) against the
   same fp64 oracle ("gate chained parity at ~2x the measured fp32 floor").  TF32
   and bf16 chained errors are reported (gpurun_out/fullsize_chained.json), not gated.
4. Every node of the chained step (all configs, including cfg5 at width 32768 where an fp64
   chain does not fit in memory): each sub_op block equals its op applied in fp64 to its stored
   source blocks, every fetch/slice/concat piece equals its source region bit for bit, every
   reduce_partial equals the ordered sum of its partials.

Stated tolerances (normwise), per op:  3xTF32 <= 2e-6, TF32 <= 2e-3, bf16 <= 1e-2;
elementwise on stored inputs: fp32 <= 1e-6, bf16 <= 8e-3; copies: bit-exact.
"""
import gzip
import json
import os

import pytest

from tests.devview import get, normwise, put

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
TOL_OP = {1: 2e-6, 0: 2e-3, "bf16": 1e-2}
TOL_EW = {4: 1e-6, 2: 8e-3}

EPI_TANH, EPI_DTANH, EPI_SCALE, EPI_SUB_OP = 1, 2, 3, 6


def plan_text(name, mode="opt", k=0):
    return gzip.open(os.path.join(ROOT, "plans", f"{name}.{mode}.k{k}.plan.json.gz"), "rt").read()


def _record(name, key, value):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name)
    d = {}
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
    d[key] = value
    with open(path, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "GPU test needs a CUDA device"
    from paper_1805_04170_b200.executor import Context
    return Context(0)


# ------------------------------------------------------------------ 1. benched kernel variants
BENCHED = {
    # id: (M, N, K, ta, tb, epilogue ops, expected variant fields)
    "cfg2_fwd_act": (512, 8192, 8192, False, False, [EPI_TANH], {"pair": 1, "bn": 256}),
    "cfg2_fwd_act_seed": (512, 8192, 8192, False, False, [EPI_TANH, EPI_DTANH], {"pair": 1, "bn": 256}),
    "cfg2_bwd_x_dact": (512, 8192, 8192, False, True, [EPI_DTANH], {"pair": 1, "bn": 256}),
    "cfg2_bwd_w_sgd": (8192, 8192, 512, True, False, [EPI_SCALE, EPI_SUB_OP],
                       {"pair": 1, "bn": 256, "p_mn": 1, "q_mn": 1, "other_smem": 1}),
    "alexconv_bwd_a": (3456, 100352, 256, True, False, [], {"pair": 1, "bn": 256}),
}


def _bf16_stage(op, v, o):
    """One fused stage as the kernel computes it on the stored (rounded) previous value."""
    import torch
    f = v.float()
    if op == EPI_TANH:
        r = torch.tanh(f.double())
    elif op == EPI_DTANH:
        t = torch.tanh(f.double())
        r = 1 - t * t
    elif op == EPI_SCALE:
        r = (f * 0.01).double()
    else:
        r = (o.float() - f).double()
    return r


@pytest.mark.parametrize("precision", [0, 2], ids=["tf32", "bf16"])
@pytest.mark.parametrize("case", sorted(BENCHED))
def test_benched_gemm_variant(case, precision):
    import torch
    from paper_1805_04170_b200 import native
    M, N, K, ta, tb, epi, expect = BENCHED[case]
    dt = torch.bfloat16 if precision == 2 else torch.float32
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + 7 * K)
    A = (torch.rand((K, M) if ta else (M, K), device="cuda", generator=g) * 2 - 1).to(dt)
    B = (torch.rand((N, K) if tb else (K, N), device="cuda", generator=g) * 2 - 1).to(dt)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=dt)
    W = (torch.rand((M, N), device="cuda", generator=g) * 2 - 1).to(dt) if EPI_SUB_OP in epi else None
    outs = [torch.full((M, N), float("nan"), device="cuda", dtype=dt) for _ in epi]
    native.gemm(A, B, ta, tb, C, epi=[(op, 0.01, W if op == EPI_SUB_OP else None, o) for op, o in zip(epi, outs)],
                precision=precision)
    torch.cuda.synchronize()
    info = native.last_launch()
    for key, want in expect.items():
        assert info[key] == want, (case, key, info)
    if EPI_SUB_OP in epi and precision == 0:
        assert info["oloader"] == 1, info  # fp32 update epilogue: operand-loader warp
    Ad, Bd = A.double(), B.double()
    ref = (Ad.t() if ta else Ad) @ (Bd.t() if tb else Bd)
    e = normwise(C, ref)
    tol = TOL_OP["bf16"] if precision == 2 else TOL_OP[0]
    assert e <= tol, (case, "product", e)
    prev = C
    errs = {"product": e}
    for i, (op, out) in enumerate(zip(epi, outs)):
        if precision == 0 and op in (EPI_SCALE, EPI_SUB_OP):
            want = prev * 0.01 if op == EPI_SCALE else W - prev
            assert torch.equal(out, want), (case, i)  # fp32 elementwise: bit-exact
            errs[f"stage{i}"] = 0.0
        else:
            want = _bf16_stage(op, prev, W)
            e = (out.double() - want).abs().max().item() / max(want.abs().max().item(), 1e-30)
            errs[f"stage{i}"] = e
            assert e <= (TOL_EW[2] if precision == 2 else TOL_EW[4]), (case, i, e)
        prev = out
    _record("benched_gemm.json", f"{case}.{'bf16' if precision == 2 else 'tf32'}", {"launch": info, "normwise": errs})


def test_benched_pair_matches_single_cta():
    """The CTA-pair bwd_w + SGD kernel and the single-CTA kernel (debug knob (6,1)) on the same
    operands: both within the TF32 gate of fp64, within TF32 noise of each other (the pair's
    M = 256 MMAs and the single CTA's M = 128 MMAs need not round the same way)."""
    import torch
    from paper_1805_04170_b200 import native
    M, N, K = 4096, 4096, 512
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.rand((K, M), device="cuda", generator=g) * 2 - 1
    B = torch.rand((K, N), device="cuda", generator=g) * 2 - 1
    W = torch.rand((M, N), device="cuda", generator=g) * 2 - 1
    ref = A.double().t() @ B.double()
    res = []
    for no_pair in (0, 1):
        native.lib().tpx_debug_gemm_mn_desc(6, no_pair)
        try:
            C, wd, wn = (torch.empty((M, N), device="cuda") for _ in range(3))
            native.gemm(A, B, True, False, C, epi=[(EPI_SCALE, 0.01, None, wd), (EPI_SUB_OP, 0.0, W, wn)])
            torch.cuda.synchronize()
            assert native.last_launch()["pair"] == 1 - no_pair
            assert normwise(C, ref) <= TOL_OP[0]
            assert torch.equal(wd, C * 0.01) and torch.equal(wn, W - wd)
            res.append(C)
        finally:
            native.lib().tpx_debug_gemm_mn_desc(6, 0)
    assert normwise(res[0], res[1].double()) <= 1e-3


# ------------------------------------------------------------------ 2./3. whole plans at full size
FULL = [  # (plan name, k): the benched workloads (bench.py CONFIGS), tiled on one GPU for k > 0
    ("cfg2_mlp5x8192_b512", 0), ("cfg2_mlp5x8192_b512", 3), ("alexfc_b128", 0), ("alexfc_b128", 3),
    ("vggfc_b64", 0), ("alexconv_b128", 0), ("vggconv_b64", 0), ("alexconv_b128", 2),
]
_oracle_cache = {}


def oracle_nodes(name, k, mode="opt"):
    """fp64 value of every node (torch restatement of execute_numeric, on the GPU)."""
    from oracle import torch_oracle as T
    key = (name, k, mode)
    if key not in _oracle_cache:
        _oracle_cache.clear()
        import torch
        torch.cuda.empty_cache()
        text = plan_text(name, mode, k)
        P = json.loads(text)
        serial = T.serial_execute(P["graph"], 7, device="cuda")
        _oracle_cache[key] = (text, P, serial, T.execute_nodes(P, serial))
    return _oracle_cache[key]


def compute_ops(ex):
    return {s["op"] for s in ex.describe()["main"]["steps"]
            if s["kind"] in ("gemm", "conv") or s["what"] == "elementwise"}


def _tf32(x):
    """An fp32 operand as a kind::tf32 MMA reads it: the low 13 mantissa bits are ignored
    (truncation toward zero to 10 explicit mantissa bits)."""
    import torch
    i = x.float().contiguous().view(torch.int32)
    return (i & ~0x1FFF).view(torch.float32).double()


def _floor_out(op, ins, prec):
    """The op on teacher-forced inputs as the kernel can represent them, computed to the
    precision floor: TF32 operands in fp64 (tf32), fp32 inputs in IEEE fp32 arithmetic
    (3xTF32's target), bf16 inputs in fp64 (bf16)."""
    import torch
    from oracle import torch_oracle as T
    mm = op["kind"] in ("matmul", "conv")
    if prec == "bf16":
        return T.run_op_dense(op, [x.float().to(torch.bfloat16).double() for x in ins])
    if prec == 0 and mm:
        return T.run_op_dense(op, [_tf32(x) for x in ins])
    if prec == 1 and mm:
        tf = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
        torch.backends.cuda.matmul.allow_tf32 = torch.backends.cudnn.allow_tf32 = False
        try:
            return T.run_op_dense(op, [x.float() for x in ins]).double()
        finally:
            torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = tf
    return T.run_op_dense(op, [x.float().double() for x in ins])


# per-op gates: err <= A * floor + B, floor = the precision floor on the same inputs (_floor_out)
GATE = {0: (2.0, 1e-5), 1: (2.0, 1e-6), "bf16": (1.5, 4e-3)}


def run_teacher_forced(ctx, name, k, precision):
    """Per op: oracle inputs in, that op's lowered steps, outputs compared.  Returns
    {op: (error, floor, own steps, kind)} (fused ops: vs the op on the stored inputs, floor 0)."""
    from oracle import torch_oracle as T
    from paper_1805_04170_b200.executor import FLAG_FUSE, PlanExecutor
    text, P, serial, vals = oracle_nodes(name, k)
    if precision == "bf16":
        bP = json.loads(plan_text(name + "_bf16", "opt", k))
        assert [n["region"] for n in bP["nodes"]] == [n["region"] for n in P["nodes"]]
        text, P = json.dumps(bP), bP
    ex = PlanExecutor(ctx, text, precision=0 if precision == "bf16" else precision, flags=FLAG_FUSE)
    ex.init_inputs(7)
    own = compute_ops(ex)
    errs = {}
    for op in P["graph"]["ops"]:
        subs = [n for n in P["nodes"] if n["kind"] == "sub_op" and n["op"] == op["id"]]
        if op["id"] in own:
            for t in op["inputs"]:
                for h in P["holders"][t]:
                    put(ex, h, vals[h])
        ex.execute_op(op["id"])
        ex.synchronize()
        if op["id"] in own:
            e = max(normwise(get(ex, h), vals[h]) for h in P["holders"][op["output"]])
            fl = max(normwise(_floor_out(op, [vals[s] for s in n["sources"]], precision), vals[n["id"]]) for n in subs)
        else:
            e = max(normwise(get(ex, n["id"]), T.run_op_dense(op, [get(ex, s) for s in n["sources"]])) for n in subs)
            fl = 0.0
        errs[op["id"]] = (e, fl, op["id"] in own, op["kind"])
    ex.close()
    return errs


@pytest.mark.parametrize("precision", [0, 1, "bf16"], ids=["tf32", "fp32", "bf16"])
@pytest.mark.parametrize("name,k", FULL, ids=lambda x: str(x))
def test_fullsize_per_op(ctx, name, k, precision):
    if precision == "bf16" and not os.path.exists(os.path.join(ROOT, "plans", f"{name}_bf16.opt.k{k}.plan.json.gz")):
        pytest.skip("no bf16 plan for this config")
    errs = run_teacher_forced(ctx, name, k, precision)
    key = {0: "tf32", 1: "fp32", "bf16": "bf16"}[precision]
    _record("fullsize_per_op.json", f"{name}.k{k}.{key}", {op: {"err": e, "floor": f} for op, (e, f, _, _) in errs.items()})
    a, b = GATE[precision]
    for op, (e, fl, own, kind) in errs.items():
        if own:
            tol = a * fl + (b if kind != "elementwise" else TOL_EW[2 if precision == "bf16" else 4])
        else:
            tol = TOL_EW[2 if precision == "bf16" else 4]
        assert e <= tol, (op, e, fl, tol)


def chained_errors(ctx, text, P, serial, vals, precision):
    from paper_1805_04170_b200.executor import FLAG_FUSE, FLAG_GRAPH, PlanExecutor
    ex = PlanExecutor(ctx, text, precision=precision, flags=FLAG_FUSE | FLAG_GRAPH)
    ex.init_inputs(7)
    ex.execute()
    ex.synchronize()
    per_t = {}
    for t, hs in P["holders"].items():
        per_t[t] = max(normwise(get(ex, h), vals[h]) for h in hs)
    ex.close()
    return per_t


@pytest.mark.parametrize("name,k", [("cfg2_mlp5x8192_b512", 0), ("cfg2_mlp5x8192_b512", 3), ("alexfc_b128", 0),
                                    ("vggfc_b64", 2), ("alexconv_b128", 0), ("vggconv_b64", 1)], ids=lambda x: str(x))
def test_fullsize_chained(ctx, name, k):
    import torch
    from oracle import torch_oracle as T
    text, P, serial, vals = oracle_nodes(name, k)
    tf = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = torch.backends.cudnn.allow_tf32 = False
    try:
        floor_vals = T.serial_execute(P["graph"], 7, device="cuda", dtype=torch.float32)
    finally:
        torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = tf
    floor = {t: normwise(floor_vals[t], serial[t]) for t in P["holders"]}
    del floor_vals
    ours = chained_errors(ctx, text, P, serial, vals, 1)
    tf32 = chained_errors(ctx, text, P, serial, vals, 0)
    rec = {"fp32_floor_worst": max(floor.values()), "ours_3xtf32_worst": max(ours.values()),
           "ours_tf32_worst": max(tf32.values()),
           "per_tensor": {t: {"floor": floor[t], "3xtf32": ours[t], "tf32": tf32[t]} for t in floor}}
    try:
        bP = json.loads(plan_text(name + "_bf16", "opt", k))
        rec["ours_bf16_worst"] = max(chained_errors(ctx, json.dumps(bP), bP, serial, vals, 0).values())
    except FileNotFoundError:
        pass
    _record("fullsize_chained.json", f"{name}.k{k}", rec)
    worst_floor = max(floor.values())
    if worst_floor > 0.1:
        # the chain has no significant digits even in plain fp32 (structural
        # 1 - tanh^2 on unscaled inputs); per-op parity carries the check, the errors are recorded
        pytest.skip(f"ill-conditioned at full size: fp32 floor {worst_floor:.3g} (recorded)")
    assert rec["ours_3xtf32_worst"] <= 2 * worst_floor + 1e-6, rec["ours_3xtf32_worst"]


# ------------------------------------------------------------------ 4. every node, all configs
SELF = [("cfg2_mlp5x8192_b512", 0, 0), ("cfg2_mlp5x8192_b512", 3, 0), ("cfg2_mlp5x8192_b512_bf16", 0, 0),
        ("cfg5_mlp3x32768_b32", 0, 0), ("cfg5_mlp3x32768_b32", 1, 0), ("cfg5_mlp3x32768_b32_bf16", 0, 0),
        ("alexfc_b128", 2, 0), ("vggfc_b64", 0, 0), ("alexconv_b128", 0, 0), ("vggconv_b64", 0, 0),
        ("alexconv_b128_bf16", 0, 0), ("cfg2_mlp5x8192_b512", 0, 1)]


@pytest.mark.parametrize("name,k,precision", SELF, ids=lambda x: str(x))
def test_fullsize_every_node(ctx, name, k, precision):
    import torch
    from oracle import torch_oracle as T
    from paper_1805_04170_b200.executor import FLAG_FUSE, FLAG_GRAPH, PlanExecutor
    _oracle_cache.clear()
    torch.cuda.empty_cache()
    text = plan_text(name, "opt", k)
    P = json.loads(text)
    ex = PlanExecutor(ctx, text, precision=precision, flags=FLAG_FUSE | FLAG_GRAPH)
    bf = ex.storage_bytes() == 2
    ex.init_inputs(7)
    ex.execute()
    ex.synchronize()
    ops = {o["id"]: o for o in P["graph"]["ops"]}
    nodes = {n["id"]: n for n in P["nodes"]}
    worst = {}
    for n in P["nodes"]:
        kind = n["kind"]
        if kind == "buffer":
            continue
        if kind in ("fetch", "slice"):
            s = nodes[n["sources"][0]]
            try:
                got = get(ex, n["id"])
            except Exception:  # a piece written straight into its concat holds no value of its own
                continue
            sl = tuple(slice(lo - s0, hi - s0) for (lo, hi), (s0, _) in zip(n["region"], s["region"]))
            assert torch.equal(got, get(ex, s["id"])[sl]), n["id"]
            continue
        got = get(ex, n["id"])
        if kind == "concat":
            for s in n["sources"]:
                sn = nodes[s]
                sl = tuple(slice(lo - c0, hi - c0) for (lo, hi), (c0, _) in zip(sn["region"], n["region"]))
                src = get(ex, s) if _has(ex, s) else None
                if src is not None:
                    assert torch.equal(got[sl], src), (n["id"], s)
            continue
        if kind == "reduce_partial":
            # a fetched partial read in place by the reduction holds no value of its own: its
            # source region stands in for it
            want = sum(get(ex, s) if _has(ex, s) else _region_of(ex, nodes, s) for s in n["sources"])
            e, key = normwise(got, want), "reduce_partial"
        else:
            op = ops[n["op"]]
            want = T.run_op_dense(op, [get(ex, s) for s in n["sources"]])
            e, key = normwise(got, want), n["op"]
            key = op["kind"] if op["kind"] != "elementwise" else op["attrs"]["function"]
        worst[key] = max(worst.get(key, 0.0), e)
    ex.close()
    _record("fullsize_every_node.json", f"{name}.k{k}.p{precision}", worst)
    for key, e in worst.items():
        if key in ("matmul", "conv"):
            tol = TOL_OP["bf16"] if bf else TOL_OP[precision]
        else:
            tol = TOL_EW[2] if bf else TOL_EW[4]
        assert e <= tol, (key, e, tol)


def _region_of(ex, nodes, node_id):
    n = nodes[node_id]
    s = nodes[n["sources"][0]]
    sl = tuple(slice(lo - s0, hi - s0) for (lo, hi), (s0, _) in zip(n["region"], s["region"]))
    return get(ex, s["id"])[sl]


def _has(ex, node_id):
    try:
        ex.node_view(node_id)
        return True
    except Exception:
        return False
