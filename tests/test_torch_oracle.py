"""Pins the torch fp64 restatement (oracle/torch_oracle.py, used by the full-size GPU parity
tests) to the reference: the golden fixtures produced by the compiled reference's own node loop
(tools/make_golden.py), on CPU.  Same gates as the numpy restatement (test_oracle.py):
seeded inputs bit-exact, every node value within 1e-10 of the reference's (summation order)."""
import numpy as np
import pytest
import torch

from oracle import tileplan_oracle as O
from oracle import torch_oracle as T
from tests.conftest import golden_stems, load_golden, stem_id, summary

STEMS = [s for s in golden_stems() if any(k in stem_id(s) for k in
                                          ("cfg2r_mlp5x256_b64.opt", "alexr_conv_b4.opt", "cnn_train",
                                           "reduce_kat", "fcr_alexnet_b32.data", "wideconv_b2",
                                           "mlp_train_d4.hybrid"))]


def test_inventory():
    assert len(STEMS) >= 10


@pytest.mark.parametrize("shape,seed,tid", [((7, 13), 7, "w1"), ((3, 4, 5, 6), 33, "a0"), ((100003,), 5, "x0")])
def test_seeded_tensor_bit_exact(shape, seed, tid):
    got = T.seeded_tensor(shape, seed, tid, chunk=4096).numpy()
    want = O.seeded_tensor(shape, seed, tid)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("stem", STEMS, ids=stem_id)
def test_torch_oracle_matches_reference_golden(stem):
    _, P, vals, seed = load_golden(stem)
    serial = T.serial_execute(P["graph"], seed)
    nodes = T.execute_nodes(P, serial)
    for key, want in vals.items():
        kind, name = key.split(":", 1)
        got = (nodes[name] if kind != "serial" else serial[name]).numpy()
        if kind == "summary":
            got = summary(got)
            scale = np.array([want[1], want[1], want[2]])
            assert (np.abs(got[:3] - want[:3]) <= 1e-11 * np.maximum(scale, 1.0)).all(), key
            got, want = got[3:], want[3:]
        assert got.shape == want.shape, key
        d = np.abs(got - want)
        rel = float((d / np.maximum(np.abs(want), 1.0)).max()) if d.size else 0.0
        assert rel <= 1e-10, (key, rel)


def test_fp32_floor_mode():
    """dtype=float32 runs the same graph in plain fp32 (the floor the chained gates cite)."""
    _, P, _, seed = load_golden(STEMS[0])
    a = T.serial_execute(P["graph"], seed)
    b = T.serial_execute(P["graph"], seed, dtype=torch.float32)
    for t in a:
        assert b[t].dtype == torch.float32
        err = (b[t].double() - a[t]).abs().max() / a[t].abs().max().clamp_min(1e-30)
        assert err < 0.1, t
