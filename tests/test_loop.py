"""Training loop: repeated steps with the weights carried from w_next into w (SURVEY §8(f) rank 1,
§7 H1; reference: gen_mlp leaves w<l>_next dangling, proj/src/graph.cpp:217-227, and graph
inputs start resident at no cost, proj/src/execgraph.cpp:196-213, so the planner prices one
step and never the carry).

TPX_FLAG_LOOP lowers the step twice; weights whose w_next holder has the weight's own layout
on every device trade storage between the two programs, so the carry is free (data-parallel
and loop-aware plans); the rest run the carry conversion after each step, and its cross-device
bytes are the "unpriced" bytes of the single-step optimum.

CPU: host-only lowering, accounting.  GPU: three loop steps equal three (step, carry) rounds bit
for bit, with and without CUDA-graph replay."""
import gzip
import json
import os

import numpy as np
import pytest

from tests.conftest import golden_stems, load_golden, stem_id

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def plan(name, mode, k):
    return gzip.open(os.path.join(ROOT, "plans", f"{name}.{mode}.k{k}.plan.json.gz"), "rt").read()


@pytest.fixture(scope="module")
def host():
    from paper_1805_04170_b200.executor import Context
    return Context.host_only()


def test_cfg2_carry_bytes_match_survey(host):
    """The single-step optimum at k=3 keeps w replicated and w_next row-split: its carry moves
    9,395,240,960 bytes across devices per step (SURVEY finding 5), none of them priced."""
    from paper_1805_04170_b200.executor import FLAG_FUSE, FLAG_LOOP, PlanExecutor
    ex = PlanExecutor(host, plan("cfg2_mlp5x8192_b512", "opt", 3), flags=FLAG_FUSE | FLAG_LOOP)
    d = ex.describe()
    assert d["loop"] == 1 and d["swapped"] == [] and d["carry_bytes"] == 9395240960
    assert len(d["carry"]["steps"]) > 0


@pytest.mark.parametrize("name,mode,k", [("cfg2_mlp5x8192_b512", "data", 3), ("cfg2_mlp5x8192_b512", "opt", 0),
                                         ("alexfc_b128", "loop", 1), ("alexconv_b128", "data", 2),
                                         ("cfg1_mlp3x1024_b64", "data", 1)])
def test_loop_consistent_plans_swap(host, name, mode, k):
    """Data-parallel (w, w_next both r^k), k = 0 and loop-aware plans carry by the swap alone: no
    carry program, no extra arena, the same per-op bytes as the single program."""
    from paper_1805_04170_b200.executor import FLAG_FUSE, FLAG_LOOP, PlanExecutor
    text = plan(name, mode, k)
    a = PlanExecutor(host, text, flags=FLAG_FUSE)
    b = PlanExecutor(host, text, flags=FLAG_FUSE | FLAG_LOOP)
    da, db = a.describe(), b.describe()
    weights = sorted(t["id"][:-5] for t in json.loads(text)["graph"]["tensors"] if t["id"].endswith("_next"))
    assert sorted(db["swapped"]) == weights
    assert db["carry"]["steps"] == [] and db["carry_bytes"] == 0
    assert a.stats()["device_bytes"] == b.stats()["device_bytes"]
    assert da["per_op_fetch_bytes_in"] == db["per_op_fetch_bytes_in"]
    assert [s["op"] for s in da["main"]["steps"]] == [s["op"] for s in db["main"]["steps"]]


STEMS = [s for s in golden_stems() if any(k in stem_id(s) for k in
                                          ("cfg2r_mlp5x256_b64.opt.k2", "cfg2r_mlp5x256_b64.data.k2",
                                           "mlp_train_d3.opt.k1", "cfg1_bf16.opt.k1", "alexr_conv_b4.data.k1",
                                           "fcr_alexnet_b32.opt.k3"))]


@pytest.mark.gpu
@pytest.mark.parametrize("graph", [0, 1], ids=["eager", "graph"])
@pytest.mark.parametrize("stem", STEMS, ids=stem_id)
def test_loop_steps_match_step_then_carry(stem, graph):
    from paper_1805_04170_b200.executor import FLAG_FUSE, FLAG_GRAPH, FLAG_LOOP, Context, PlanExecutor
    text, P, _, seed = load_golden(stem)
    ctx = Context(0)
    fl = FLAG_FUSE | (FLAG_GRAPH if graph else 0)
    prec = 0 if "bf16" in stem else 1
    a = PlanExecutor(ctx, text, precision=prec, flags=fl)
    b = PlanExecutor(ctx, text, precision=prec, flags=fl | FLAG_LOOP)
    a.init_inputs(seed)
    b.init_inputs(seed)
    for _ in range(3):
        a.execute()
        a.carry_weights()
        b.execute()
    a.synchronize()
    b.synchronize()
    for t, hs in P["holders"].items():
        if t.endswith("_next") or t + "_next" in P["holders"]:
            continue  # a's weights were overwritten by its last carry; b's hold this step's inputs
        for h in hs:
            assert np.array_equal(a.read_node(h), b.read_node(h)), (t, h)
    for t in P["holders"]:
        if t.endswith("_next"):
            for h in P["holders"][t]:
                assert np.array_equal(a.read_node(h), b.read_node(h)), (t, h)
    a.close()
    b.close()
