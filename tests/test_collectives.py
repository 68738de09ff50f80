"""Collective classification of plan phases (paper_1805_04170_b200/collectives.py), on the benched
plans and the SURVEY §8(e) expectations: the cfg2 optimum gathers g (AllGather, 8 devices) and
re-partitions x (AllToAll) for every bwd_w; the data preset adds the w_next AllGather of every
update; the AlexNet-style conv data plan reduce-scatters every filter gradient; the group bits are
the cut bits of the conversion (device id = cut bits, proj/src/tiling.cpp:200-210)."""
import gzip
import json
import os

from paper_1805_04170_b200.collectives import classify_phases, describe_collectives

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def plan(name):
    return json.loads(gzip.open(os.path.join(ROOT, "plans", name + ".plan.json.gz")).read())


def test_cfg2_opt_k3():
    P = plan("cfg2_mlp5x8192_b512.opt.k3")
    ph = {p["phase"]: p for p in classify_phases(P)}
    for l in (2, 3, 4, 5):
        assert ph[f"bwd_w{l}:in1"]["pattern"] == "all_gather"
        assert ph[f"bwd_w{l}:in1"]["group_sizes"] == [8] and ph[f"bwd_w{l}:in1"]["cut_bits"] == 7
        assert ph[f"bwd_w{l}:in0"]["pattern"] == "all_to_all"
    tot = describe_collectives(P)
    assert sum(t["bytes"] for t in tot.values()) == P["fetch_bytes_total"]


def test_cfg2_data_adds_update_all_gather():
    P = plan("cfg2_mlp5x8192_b512.data.k3")
    ph = {p["phase"]: p for p in classify_phases(P)}
    for l in range(1, 6):
        assert ph[f"upd{l}:out"]["pattern"] == "all_gather"
    assert sum(p["bytes"] for p in ph.values()) == P["fetch_bytes_total"]


def test_conv_data_reduce_scatter_and_loop_groups():
    P = plan("alexconv_b128.data.k2")
    ph = {p["phase"]: p for p in classify_phases(P)}
    for l in range(1, 6):
        assert ph[f"bwd_k{l}:out"]["pattern"] == "reduce_scatter"
        assert ph[f"bwd_k{l}:out"]["group_sizes"] == [4]
    L = plan("cfg2_mlp5x8192_b512.loop.k3")
    pats = {p["pattern"] for p in classify_phases(L)}
    assert "reduce_scatter" in pats
    # loop-consistent hybrids communicate inside bit-subset groups smaller than the whole job
    assert any(p["group_sizes"] != [8] for p in classify_phases(L))
