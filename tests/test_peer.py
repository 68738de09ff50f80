"""Peer-pull exchange (TPX_FLAG_PEER, csrc/runtime.cpp): host-only lowering checks on CPU.

In peer mode a cross-rank fetch (`fetch` node whose source device lives on another rank,
reference: proj/src/simulator.cpp:88-93, pieces from Builder::assemble,
proj/src/execgraph.cpp:101-188) is executed by the CONSUMING rank as one pull launch per phase
that reads the strided box out of the owner's arena over NVLink.  These tests lower every golden
plan for every rank of a 2-rank and a 2^k-rank job and check:
  * the byte contract is unchanged: per-op fetch bytes == graph_cost per_op, and the bytes each
    rank pulls from other ranks == the plan's fetch bytes whose source lives on another rank;
  * every rank runs the SAME sequence of sync points (signals per phase with a cross-rank fetch,
    one closing barrier), the invariant the device-side counters rely on;
  * no NCCL group is left, and a pull only waits on ranks other than its own;
  * partials consumed by a reduce_partial are read in place (no copy of their own) and the
    reduction carries its elementwise consumers (SGD step + update) when they follow it.
"""
import json

import pytest

from oracle import tileplan_oracle as O
from paper_1805_04170_b200.executor import FLAG_FORCE_XCHG, FLAG_FUSE, FLAG_LOOP, FLAG_PEER, Context, PlanExecutor
from tests.conftest import golden_stems, load_golden, stem_id

STEMS = golden_stems()
MULTI = [s for s in STEMS if int(stem_id(s).split(".k")[1].split(".")[0]) >= 1]


def sync_sequence(desc, prog="main"):
    """Sync points in launch order: a signal folded into a phase's first conversion launch or a
    one-thread signal launch (its index), or a barrier ("B")."""
    out = []
    for s in desc[prog]["steps"]:
        if s["kind"] == "sync":
            out.append("B" if s["barrier"] else s["signal"])
        elif s["kind"] == "nary" and s.get("signal", -1) >= 0:
            out.append(s["signal"])
    return out


@pytest.mark.parametrize("stem", MULTI, ids=stem_id)
def test_peer_lowering_bytes_and_sync(stem):
    text, P, _, _ = load_golden(stem)
    per_op = O.per_op_bytes(P)
    for world in sorted({2, P["devices"]}):
        exs = [PlanExecutor(Context.host_only(r, world), text, flags=FLAG_FUSE | FLAG_PEER) for r in range(world)]
        descs = [e.describe() for e in exs]
        stats = [e.stats() for e in exs]
        dev_rank = lambda d: (d * world) // P["devices"]  # noqa: E731
        cross_in = [0] * world
        for n in P["nodes"]:
            if n["kind"] == "fetch" and dev_rank(n["device"]) != dev_rank(n["src_device"]):
                cross_in[dev_rank(n["device"])] += n["bytes"]
        assert [d["pull_bytes_in"] for d in descs] == cross_in
        assert [s["rank_xrank_bytes_in"] for s in stats] == cross_in
        assert sum(s["rank_fetch_bytes_in"] for s in stats) == P["fetch_bytes_total"]
        tot = {}
        for d in descs:
            for k, v in d["per_op_fetch_bytes_in"].items():
                tot[k] = tot.get(k, 0) + v
        assert tot == per_op
        seqs = [sync_sequence(d) for d in descs]
        assert all(q == seqs[0] for q in seqs), "ranks disagree on the sync points"
        xphases = {n["phase"] for n in P["nodes"]
                   if n["kind"] == "fetch" and dev_rank(n["device"]) != dev_rank(n["src_device"])}
        assert seqs[0] == (list(range(len(xphases))) + ["B"] if xphases else [])
        for r, d in enumerate(descs):  # every pull waits for its own phase's sync point
            for s in d["main"]["steps"]:
                if s["kind"] == "nary" and s.get("pull"):
                    assert 0 <= s["wait_s"] < len(xphases)
        for r, d in enumerate(descs):
            steps = d["main"]["steps"]
            assert not [s for s in steps if s["kind"] == "nccl"]
            for s in steps:
                if s["kind"] == "nary" and s.get("pull"):
                    assert not (s["wait_mask"] >> r) & 1, "a pull waits on its own rank"
            if cross_in[r]:
                assert any(s["kind"] == "nary" and s.get("pull") for s in steps)


@pytest.mark.parametrize("stem", [s for s in MULTI if ".k1." in s][:8], ids=stem_id)
def test_peer_forced_single_rank(stem):
    """world 1 + FORCE_XCHG + PEER: every cross-device fetch is a pull against the rank's own
    arena (the single-GPU exercise of the peer path): bytes unchanged, no NCCL."""
    text, P, _, _ = load_golden(stem)
    ex = PlanExecutor(Context.host_only(), text, flags=FLAG_FUSE | FLAG_FORCE_XCHG | FLAG_PEER)
    d, st = ex.describe(), ex.stats()
    assert st["rank_fetch_bytes_in"] == P["fetch_bytes_total"]
    assert st["n_nccl_groups"] == 0
    if P["fetch_bytes_total"]:
        assert d["sync_points"] >= 2


REDUCE_SGD = [s for s in STEMS if stem_id(s).startswith(("mlp_train_d2.data.k", "alexr_conv_b4.data.k1",
                                                             "mlp_train_d3.opt.k2"))]


@pytest.mark.parametrize("stem", REDUCE_SGD, ids=stem_id)
def test_peer_reduce_reads_partials_in_place_and_fuses_sgd(stem):
    """grad_weight in the reduce form: every reduce_partial reads its fetched partials where they
    lie and the SGD step + update of the reduced gradient run in the same launch (the unfused
    lowering would leave a step / upd elementwise launch)."""
    text, P, _, _ = load_golden(stem)
    reduces = [n for n in P["nodes"] if n["kind"] == "reduce_partial"]
    assert reduces
    for flags, world in ((FLAG_FUSE, 1), (FLAG_FUSE | FLAG_PEER, 2)):
        for r in range(world):
            ex = PlanExecutor(Context.host_only(r, world), text, flags=flags)
            steps = ex.describe()["main"]["steps"]
            red = [s for s in steps if s["kind"] == "nary" and s["what"] == "reduce"]
            assert red and sum(s["chained"] for s in red) > 0
            ew_ops = {s["op"] for s in steps if s["kind"] == "nary" and s["what"] == "elementwise"}
            assert not {o for o in ew_ops if o.startswith(("step", "upd"))}, ew_ops
            # no copy step materialises a fetched partial that only the reduction reads
            cons = {}
            for n in P["nodes"]:
                for s in n.get("sources", []):
                    cons.setdefault(s, []).append(n)
            fetched = [n for n in P["nodes"] if n["kind"] == "fetch" and len(cons.get(n["id"], [])) == 1
                       and cons[n["id"]][0]["kind"] == "reduce_partial"
                       and (n["device"] * world) // P["devices"] == r]
            with pytest.raises(Exception):
                if fetched:
                    ex.node_view(fetched[0]["id"])
                else:
                    raise RuntimeError("nothing fetched")


@pytest.mark.parametrize("stem", [s for s in MULTI if "mlp_train" in s and ".opt.k2." in s][:2], ids=stem_id)
def test_peer_loop_mode_carry_has_barrier(stem):
    text, P, _, _ = load_golden(stem)
    world = 2
    descs = [PlanExecutor(Context.host_only(r, world), text,
                          flags=FLAG_FUSE | FLAG_PEER | FLAG_LOOP).describe() for r in range(world)]
    carry = [sync_sequence(d, "carry") for d in descs]
    assert carry[0] == carry[1]
    if any(s["kind"] == "nary" and s.get("pull") for d in descs for s in d["carry"]["steps"]):
        assert carry[0] == ["B"]  # the carry's pulls wait for the main program's barrier
        assert all(s["wait_s"] == -1 for d in descs for s in d["carry"]["steps"] if s["kind"] == "nary" and s.get("pull"))
