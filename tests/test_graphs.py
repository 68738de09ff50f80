"""Host graph generators (paper_1805_04170_b200/graphs.py) against the reference's gen_cnn.

CPU only.  With one filter size and no update, conv_net must emit exactly gen_cnn's graph
(proj/src/graph.cpp:231-314, through oracle/_ref); with the update it must add gen_mlp's
step/upd pattern; the AlexNet/VGG presets must end at the FC components' widths."""
import json

import pytest

from paper_1805_04170_b200 import graphs as G

ref = pytest.importorskip("oracle.ref")


@pytest.fixture(scope="module")
def reflib():
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref


@pytest.mark.parametrize("args", [(8, (6, 6), [2, 4]), (16, (10, 10), [4, 8, 8]), (2, (9, 7), [3, 5, 4, 2])])
def test_conv_net_equals_gen_cnn(reflib, args):
    b, hw, ch = args
    want = json.loads(reflib.gen_cnn(b, hw, ch, (3, 3), backward=True))
    got = json.loads(G.conv_net(b, hw, ch, [(3, 3)] * (len(ch) - 1), backward=True, update=False))
    assert got == want
    want = json.loads(reflib.gen_cnn(b, hw, ch, (3, 3), backward=False))
    got = json.loads(G.conv_net(b, hw, ch, [(3, 3)] * (len(ch) - 1), backward=False, update=False))
    assert got == want


def test_update_ops_follow_gen_mlp(reflib):
    g = json.loads(G.conv_net(2, (8, 8), [2, 3, 4], [(3, 3), (2, 2)]))
    mlp = json.loads(reflib.gen_mlp(2, [4, 4, 4]))
    ups = [o for o in g["ops"] if o["id"].startswith(("step", "upd"))]
    mups = [o for o in mlp["ops"] if o["id"].startswith(("step", "upd"))]
    assert [(o["kind"], o["attrs"]) for o in ups] == [(o["kind"], o["attrs"]) for o in mups]
    assert [o["inputs"] for o in ups] == [["gk1"], ["k1", "kd1"], ["gk2"], ["k2", "kd2"]]
    roles = {t["id"]: t["role"] for t in g["tensors"]}
    assert roles["k1_next"] == "weight" and roles["kd2"] == "temp"


def test_presets_shapes():
    """VGG-style ends at the FC component's 25088 = 512 x 7 x 7; AlexNet-style (no pooling in
    the IR) ends at 256 x 28 x 28 and keeps the reference FC6 width 9216 as its own component."""
    def last(gj):
        g = json.loads(gj)
        L = max(int(t["id"][1:]) for t in g["tensors"] if t["id"][0] == "k" and t["id"][1:].isdigit())
        return next(t for t in g["tensors"] if t["id"] == f"a{L}")["shape"]
    a = last(G.vgg_conv(2))
    assert a[1] * a[2] * a[3] == G.VGG_FC[0]
    assert last(G.alexnet_conv(2))[1:] == [256, 28, 28]
    assert G.conv_flops(G.alexnet_conv(2)) > 0


def test_plannable(reflib):
    gj = G.conv_net(4, (16, 16), [3, 8, 16, 8], [(5, 5), (3, 3), (3, 3)])
    for k in (0, 1, 2):
        P = json.loads(reflib.plan(gj, "opt", k))
        assert P["k"] == k and P["nodes"]
