"""Pins the numpy oracle (oracle/tileplan_oracle.py) to the reference itself.

The golden fixtures in tests/golden/ were produced by the unmodified reference library
(tools/make_golden.py: gen_mlp/gen_cnn -> preset_assignment/kcuts -> build_execution_graph ->
execute_numeric's node loop, compiled from /root/reference by oracle/Makefile).  These CPU tests
check the restatement against them and against the reference's own known answers:
  acceptance.cpp:277-293 (criterion 8: numeric equivalence <= 1e-12), :257-275 (criterion 7:
  byte conservation), test_plan.cpp:178-189 (kcuts k=2, seed 17), :191-223 (reduce KAT),
  cost.cpp:244-253 (per-op bytes = fetch bytes of the op's phases).
"""
import json

import numpy as np
import pytest

from oracle import tileplan_oracle as O
from tests.conftest import golden_stems, load_golden, stem_id, summary

STEMS = golden_stems()


def test_fixture_inventory():
    assert len(STEMS) >= 98
    names = {stem_id(s).split(".")[0] for s in STEMS}
    for n in ("cfg1_mlp3x1024_b64", "cfg2r_mlp5x256_b64", "cfg5r_mlp3x512_b32", "fcr_alexnet_b32",
              "cnnr_train_b16", "reduce_kat", "mlp_train_d4", "cnn_fwd2"):
        assert n in names


@pytest.mark.parametrize("stem", STEMS, ids=stem_id)
def test_oracle_matches_reference_golden(stem):
    _, P, vals, seed = load_golden(stem)
    serial = O.serial_execute(P["graph"], seed)
    nodes = O.execute_nodes(P, serial)
    for key, want in vals.items():
        kind, name = key.split(":", 1)
        if kind == "node":
            got = nodes[name]
        elif kind == "serial":
            got = serial[name]
        else:
            got = summary(nodes[name])
        assert got.shape == want.shape, key
        if kind == "summary":
            # sum, sum|v|, sum v^2 over up to 2^23 elements: order-dependent at n*eps of sum|v|
            scale = np.array([want[1], want[1], want[2]])
            assert (np.abs(got[:3] - want[:3]) <= 1e-11 * np.maximum(scale, 1.0)).all(), key
            got, want = got[3:], want[3:]
        d = np.abs(got - want)
        rel = float((d / np.maximum(np.abs(want), 1.0)).max()) if d.size else 0.0
        # The reference's own gate is 1e-12 (main.cpp:361) between two runs with the SAME
        # summation order; the restatement sums K-long dot products in BLAS order instead of
        # the sequential p-loop (dense.cpp:79-88), so allow K*eps-level reassociation.
        assert rel <= 1e-10, (key, rel)


@pytest.mark.parametrize("stem", [s for s in STEMS if "k" in stem_id(s)], ids=stem_id)
def test_seeded_inputs_bit_exact(stem):
    """seeded_tensor (dense.cpp:30-57) is restated bit-for-bit: every graph input equals the
    reference's buffer values exactly."""
    _, P, vals, seed = load_golden(stem)
    ins = O.graph_inputs(P["graph"])
    for t in ins:
        if "serial:" + t in vals:
            shape = vals["serial:" + t].shape
            assert np.array_equal(O.seeded_tensor(shape, seed, t), vals["serial:" + t]), t


@pytest.mark.parametrize("stem", golden_stems("*.s33") + golden_stems("*.s17"), ids=stem_id)
def test_execute_numeric_criterion8(stem):
    """acceptance.cpp:277-293 / test_plan.cpp:178-189: max_rel <= 1e-12 on every holder."""
    _, P, _, seed = load_golden(stem)
    c = O.execute_numeric(P, seed)
    assert c["values"] > 0
    assert c["max_rel"] <= 1e-12


def test_reduce_kat():
    """test_plan.cpp:191-223: one reduce_partial per device with 2 sources, 64 B fetched."""
    stem = [s for s in STEMS if stem_id(s).startswith("reduce_kat")][0]
    _, P, vals, seed = load_golden(stem)
    reds = [n for n in P["nodes"] if n["kind"] == "reduce_partial"]
    assert len(reds) == 2 and all(len(n["sources"]) == 2 for n in reds)
    assert sum(n["bytes"] for n in P["nodes"] if n["kind"] == "fetch") == 64
    assert P["fetch_bytes_total"] == 64
    c = O.execute_numeric(P, seed)
    assert c["max_rel"] <= 1e-12


@pytest.mark.parametrize("stem", STEMS, ids=stem_id)
def test_byte_conservation(stem):
    """acceptance.cpp:257-275: the plan's fetch bytes equal fetch_bytes_total, and every fetch
    moves volume x dtype_bytes (execgraph.cpp:172)."""
    _, P, _, _ = load_golden(stem)
    dt = {t["id"]: t["dtype_bytes"] for t in P["graph"]["tensors"]}
    tot = 0
    for n in P["nodes"]:
        if n["kind"] == "fetch":
            assert n["bytes"] == O.region_volume(n["region"]) * dt[n["tensor"]]
            assert n["src_device"] != n["device"]
            tot += n["bytes"]
    assert tot == P["fetch_bytes_total"]


ref = pytest.importorskip("oracle.ref")


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("stem", [s for s in STEMS if ".custom." not in s], ids=stem_id)
def test_per_op_bytes_equal_planner_cost(stem):
    """SURVEY finding 4: per-op fetch bytes == graph_cost(g, a).per_op[op].bytes
    (cost.cpp:244-253), for the plan's own assignment."""
    _, P, _, _ = load_golden(stem)
    a = json.dumps({"k": P["k"], "tilings": P["assignment"]})
    cost = ref.graph_cost(json.dumps(P["graph"]), a, P["k"])
    want = {e["op"]: e["bytes"] for e in cost["per_op"]}
    assert O.per_op_bytes(P) == want
