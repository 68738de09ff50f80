"""C-ABI library (include/tpx.h) on CPU: it loads, exports every declared symbol, and lowers
every golden plan host-only (no GPU) with the byte accounting the planner predicts.

Byte contract (BASELINE north_star): the lowered program moves exactly
the plan's fetch bytes — per op equal to graph_cost(g, a).per_op[op].bytes
(proj/src/cost.cpp:244-253), per phase equal to simulate_traffic's phase totals
(proj/src/simulator.cpp:11-49) — on every rank split of the logical devices.
"""
import collections
import json
import os
import re

import pytest

from oracle import tileplan_oracle as O
from paper_1805_04170_b200 import native
from paper_1805_04170_b200.executor import Context, PlanExecutor, TpxError
from tests.conftest import ROOT, golden_stems, load_golden, stem_id

STEMS = golden_stems()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tpx.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(tpx_\w+)\s*\(", text, re.M)))


def test_library_loads(native_lib):
    assert native_lib.tpx_version() >= 1


def test_exports_every_header_symbol(native_lib):
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(native_lib, s)]
    assert not missing, missing
    # the ctypes binding declares exactly the header's entry points
    assert sorted(native.exported_symbols()) == syms


def test_errors_name_the_offender():
    ctx = Context.host_only()
    with pytest.raises(TpxError, match="malformed plan document"):
        PlanExecutor(ctx, "{not json")
    _, P, _, _ = load_golden([s for s in STEMS if "mlp_train_d1.opt.k1" in s][0])
    bad = json.loads(json.dumps(P))
    bad["nodes"][-1]["sources"] = ["n_does_not_exist"]
    with pytest.raises(TpxError, match="n_does_not_exist"):
        PlanExecutor(ctx, json.dumps(bad))
    half = json.loads(json.dumps(P))
    for t in half["graph"]["tensors"]:
        t["dtype_bytes"] = 3
    with pytest.raises(TpxError, match="bytes"):
        PlanExecutor(ctx, json.dumps(half))
    with pytest.raises(TpxError, match="precision"):
        PlanExecutor(ctx, json.dumps(P), precision=7)
    gen = json.loads(json.dumps(P))
    gen["graph"]["ops"][1]["kind"] = "generic"
    gen["graph"]["ops"][1]["attrs"] = {"batch_dim": 0}
    with pytest.raises(TpxError, match="unbound function tag"):
        PlanExecutor(ctx, json.dumps(gen))
    ex = PlanExecutor(ctx, json.dumps(P))
    with pytest.raises(TpxError, match="host-only"):
        ex.execute()
    with pytest.raises(TpxError):
        ex.read_node("nope")


@pytest.mark.parametrize("stem", STEMS, ids=stem_id)
def test_single_rank_lowering_bytes(stem):
    text, P, _, _ = load_golden(stem)
    ex = PlanExecutor(Context.host_only(), text)
    st = ex.stats()
    d = ex.describe()
    assert st["fetch_bytes_total"] == P["fetch_bytes_total"]
    assert st["rank_fetch_bytes_in"] == P["fetch_bytes_total"]
    assert st["rank_xrank_bytes_in"] == 0 and st["n_nccl_groups"] == 0
    assert d["per_op_fetch_bytes_in"] == O.per_op_bytes(P)
    assert d["per_phase_fetch_bytes_in"] == O.fetch_bytes_by_phase(P)
    # ... and equal the reference's own simulate_traffic phase totals (simulator.cpp:11-49)
    from oracle import ref
    if ref.available():
        t = ref.simulate_traffic(text)
        assert {r["phase"]: r["bytes"] for r in t["phases"] if r["bytes"]} == \
            {k: v for k, v in d["per_phase_fetch_bytes_in"].items() if v}
        assert t["total_bytes"] == P["fetch_bytes_total"]
    assert st["gemm_flops"] == sum(
        2 * _mm_flops(P, n) for n in P["nodes"] if n["kind"] == "sub_op" and _is_mm(P, n))
    assert st["n_kernel_launches"] > 0


def _is_mm(P, n):
    """Sub-ops that run as tcgen05 GEMMs: matmuls, and convolutions (im2col + GEMM)."""
    return {o["id"]: o for o in P["graph"]["ops"]}[n["op"]]["kind"] in ("matmul", "conv")


def _ext(region):
    return [hi - lo for lo, hi in region]


def _mm_flops(P, n):
    """Multiply-adds of the sub-op's GEMM formulation (csrc/runtime.cpp lower_conv_gemm for
    convolutions: forward N*O*Yo*Xo*C*U*V, grad_weight O*C*U*V*N*Yo*Xo, grad_input
    N*Yo*Xo*C*U*V*O with (Yo, Xo) the gradient's extent)."""
    ops = {o["id"]: o for o in P["graph"]["ops"]}
    nodes = {m["id"]: m for m in P["nodes"]}
    op = ops[n["op"]]
    if op["kind"] == "conv":
        a, b, o = (_ext(nodes[n["sources"][0]]["region"]), _ext(nodes[n["sources"][1]]["region"]),
                   _ext(n["region"]))
        mode = op["attrs"]["mode"]
        if mode == "forward":
            return o[0] * o[1] * o[2] * o[3] * b[1] * b[2] * b[3]
        if mode == "grad_weight":
            return o[0] * o[1] * o[2] * o[3] * a[0] * b[2] * b[3]
        return a[0] * a[2] * a[3] * b[1] * b[2] * b[3] * a[1]
    a = nodes[n["sources"][0]]["region"]
    kk = (a[0][1] - a[0][0]) if op["attrs"].get("transpose_a") else (a[1][1] - a[1][0])
    out = n["region"]
    return (out[0][1] - out[0][0]) * (out[1][1] - out[1][0]) * kk


def rank_programs(text, world, flags=1):
    exs = [PlanExecutor(Context.host_only(r, world), text, flags=flags) for r in range(world)]
    return exs, [e.describe() for e in exs]


def check_pairing(descs):
    """NCCL send/recv matching: for every rank pair, the k-th exchange group of r that talks to
    s pairs with the k-th group of s that talks to r, with r's sends equal (in order, node and
    bytes) to s's receives and vice versa."""
    world = len(descs)
    groups = [[s for s in d["main"]["steps"] if s["kind"] == "nccl"] +
              [s for s in d["carry"]["steps"] if s["kind"] == "nccl"] for d in descs]
    for r in range(world):
        for s in range(r + 1, world):
            gr = [[x for x in g["xfers"] if x["peer"] == s] for g in groups[r]]
            gs = [[x for x in g["xfers"] if x["peer"] == r] for g in groups[s]]
            gr = [g for g in gr if g]
            gs = [g for g in gs if g]
            assert len(gr) == len(gs), (r, s)
            for a, b in zip(gr, gs):
                a_send = [(x["node"], x["bytes"]) for x in a if x["send"]]
                b_recv = [(x["node"], x["bytes"]) for x in b if not x["send"]]
                a_recv = [(x["node"], x["bytes"]) for x in a if not x["send"]]
                b_send = [(x["node"], x["bytes"]) for x in b if x["send"]]
                assert [x[1] for x in a_send] == [x[1] for x in b_recv], (r, s)
                assert [x[1] for x in b_send] == [x[1] for x in a_recv], (r, s)


MULTI = [s for s in STEMS if int(stem_id(s).split(".k")[1].split(".")[0]) >= 1]


@pytest.mark.parametrize("stem", MULTI, ids=stem_id)
def test_multi_rank_lowering_bytes_and_pairing(stem):
    text, P, _, _ = load_golden(stem)
    per_op = O.per_op_bytes(P)
    cross_all = {}
    for world in sorted({2, P["devices"]}):
        exs, descs = rank_programs(text, world)
        stats = [e.stats() for e in exs]
        assert sum(s["rank_fetch_bytes_in"] for s in stats) == P["fetch_bytes_total"]
        assert sum(s["rank_xrank_bytes_in"] for s in stats) == sum(s["rank_xrank_bytes_out"] for s in stats)
        # cross-rank bytes = fetch nodes whose source device lives on another rank
        dev_rank = lambda d: (d * world) // P["devices"]  # noqa: E731
        cross = sum(n["bytes"] for n in P["nodes"] if n["kind"] == "fetch" and
                    dev_rank(n["device"]) != dev_rank(n["src_device"]))
        assert sum(s["rank_xrank_bytes_in"] for s in stats) == cross
        cross_all[world] = cross
        tot = {}
        for d in descs:
            for k, v in d["per_op_fetch_bytes_in"].items():
                tot[k] = tot.get(k, 0) + v
        assert tot == per_op
        assert sum(s["gemm_flops"] for s in stats) == pytest.approx(
            sum(2 * _mm_flops(P, n) for n in P["nodes"] if n["kind"] == "sub_op" and _is_mm(P, n)))
        check_pairing(descs)
    if P["devices"] > 1:
        # one logical device per rank: every fetch crosses a rank boundary
        assert cross_all[P["devices"]] == P["fetch_bytes_total"]


@pytest.mark.parametrize("stem", [s for s in MULTI if ".k1." in s][:6], ids=stem_id)
def test_forced_exchange_lowering(stem):
    """FORCE_XCHG routes every cross-device fetch through the NCCL path even on one rank (the
    single-GPU exercise of the multi-GPU data path): byte totals are unchanged."""
    text, P, _, _ = load_golden(stem)
    ex = PlanExecutor(Context.host_only(), text, flags=3)
    st = ex.stats()
    assert st["rank_fetch_bytes_in"] == P["fetch_bytes_total"]
    if P["fetch_bytes_total"]:
        assert st["n_nccl_groups"] >= 1


@pytest.mark.parametrize("stem", [s for s in STEMS if "conv" in s and ".k0." in s], ids=stem_id)
def test_conv_lowering_structure(stem):
    """Host-only lowering of conv plans (csrc/runtime.cpp lower_conv_gemm): every conv sub-op is
    ONE GEMM problem over all images' columns (channel-major layout, no per-image problems),
    col2im follows each grad_input, and act / seed / step+upd / dact are fused (no elementwise
    launch left in a single-device conv step)."""
    text, P, _, _ = load_golden(stem)
    ex = PlanExecutor(Context.host_only(), text, flags=1)
    steps = ex.describe()["main"]["steps"]
    ops = {o["id"]: o for o in P["graph"]["ops"]}
    conv_subops = collections.Counter(n["op"] for n in P["nodes"]
                                      if n["kind"] == "sub_op" and ops[n["op"]]["kind"] == "conv")
    gemm_probs = collections.Counter()
    for s in steps:
        if s["kind"] == "gemm" and ops[s["op"]]["kind"] == "conv":
            gemm_probs[s["op"]] += s["problems"]
    assert gemm_probs == conv_subops
    col2im = {s["op"] for s in steps if s.get("what") == "col2im"}
    assert col2im == {o for o in conv_subops if ops[o]["attrs"]["mode"] == "grad_input"}
    assert not [s for s in steps if s.get("what") == "elementwise"], "unfused elementwise launch"
    assert ex.stats()["n_fused_ew"] == sum(1 for o in P["graph"]["ops"] if o["kind"] == "elementwise")
