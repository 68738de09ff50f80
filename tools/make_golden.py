"""Generates tests/golden/ from the UNMODIFIED reference (oracle/_ref, built by oracle/Makefile
from /root/reference/proj/src).  Test infrastructure only; runs in the build container.

For every case: the graph comes from the reference's own generators (gen_mlp / gen_cnn,
proj/src/graph.cpp:179-314) or, for the reduce KAT, the graph of
proj/tests/test_plan.cpp:191-223; the assignment from preset_assignment / kcuts
(proj/src/assign.cpp:36-81, proj/src/kcuts.cpp:35-60); the plan from build_execution_graph +
export_plan (proj/src/execgraph.cpp:295-361).  Values are execute_numeric's node loop
(proj/src/simulator.cpp:77-127) run by the reference library itself (ref_driver Session).

Files per case  <name>.<mode>.k<k>.s<seed>.plan.json.gz   the plan document (wire format)
                <name>.<mode>.k<k>.s<seed>.values.npz     fp64 values:
  small plans (<= SMALL total node elements): "node:<id>" for every node and
                                              "serial:<tensor>" (serial_execute)
  larger plans: "summary:<holder id>" = [sum, sum|v|, sum v^2, v.flat[linspace(0, n-1, 61)]]
                for every holder node.

Usage: python tools/make_golden.py [--check]   (--check regenerates in memory and compares)
"""
from __future__ import annotations

import gzip
import io
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref
from paper_1805_04170_b200 import graphs as G  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
SMALL = 50_000


def summary(v: np.ndarray) -> np.ndarray:
    f = v.ravel()
    idx = np.linspace(0, f.size - 1, 61).astype(np.int64)
    return np.concatenate([[f.sum(), np.abs(f).sum(), (f * f).sum()], f[idx]])


def reduce_kat_graph() -> str:
    """proj/tests/test_plan.cpp:191-203."""
    return json.dumps({"ops": [{"attrs": {"transpose_a": False, "transpose_b": False}, "id": "mm",
                                "inputs": ["x", "w"], "kind": "matmul", "output": "z"}],
                       "tensors": [{"dtype_bytes": 4, "id": "w", "role": "weight", "shape": [4, 4]},
                                   {"dtype_bytes": 4, "id": "x", "role": "input", "shape": [4, 4]},
                                   {"dtype_bytes": 4, "id": "z", "role": "activation", "shape": [4, 4]}]})


def graphs() -> dict:
    """Corpus graphs (proj/tests/corpus.hpp:58-103) and reduced BASELINE configs (same
    structure as cfg1/cfg2/cfg5/AlexNet-FC/conv, smaller extents so the fp64 reference
    finishes in seconds)."""
    g = {}
    for d in (1, 2, 3, 4):  # corpus.hpp:58-69 (train MLPs, width 8, batch 8)
        g[f"mlp_train_d{d}"] = ref.gen_mlp(8, [8] * (d + 1))
    g["mlp_fwd"] = ref.gen_mlp(16, [8, 8, 8], backward=False, update=False)     # corpus.hpp:70-76
    g["mlp_rect"] = ref.gen_mlp(8, [8, 16, 8], update=False)                            # corpus.hpp:78-86
    g["cnn_train"] = ref.gen_cnn(8, (6, 6), [2, 4], (3, 3), backward=True)      # corpus.hpp:90-95
    g["cnn_fwd2"] = ref.gen_cnn(16, (8, 8), [4, 4, 8], (3, 3), backward=False)  # corpus.hpp:96-101
    g["cfg1_mlp3x1024_b64"] = ref.gen_mlp(64, [1024] * 4)     # BASELINE configs[0], full size
    g["cfg2r_mlp5x256_b64"] = ref.gen_mlp(64, [256] * 6)      # configs[1] structure, reduced
    g["cfg5r_mlp3x512_b32"] = ref.gen_mlp(32, [512] * 4)      # configs[4] structure, reduced
    g["fcr_alexnet_b32"] = ref.gen_mlp(32, [576, 256, 256, 64])  # AlexNet FC6-8 structure
    g["cnnr_train_b16"] = ref.gen_cnn(16, (10, 10), [4, 8, 8], (3, 3), backward=True)
    # AlexNet-style conv component (per-layer filters + SGD update; paper_1805_04170_b200/graphs.py)
    g["alexr_conv_b4"] = G.conv_net(4, (16, 16), [3, 8, 16, 8], [(5, 5), (3, 3), (3, 3)])
    # bf16 storage (dtype_bytes 2): same structures, the planner's bytes halve; the reference's
    # fp64 values are dtype-independent
    g["cfg1_bf16"] = ref.gen_mlp(64, [1024] * 4, dtype_bytes=2)
    g["cfg2r_bf16"] = ref.gen_mlp(64, [256] * 6, dtype_bytes=2)
    g["mlp_train_d2_bf16"] = ref.gen_mlp(8, [8] * 3, dtype_bytes=2)
    g["fcr_alexnet_bf16"] = ref.gen_mlp(32, [576, 256, 256, 64], dtype_bytes=2)
    # wide channels: the implicit-GEMM grad_input (h channels >= 128), 3x3 and 5x5 taps
    g["wideconv_b2"] = G.conv_net(2, (12, 12), [3, 16, 128, 144], [(3, 3), (3, 3), (5, 5)])
    g["wideconv_bf16"] = G.conv_net(2, (12, 12), [3, 16, 128, 144], [(3, 3), (3, 3), (5, 5)], dtype_bytes=2)
    g["alexr_conv_bf16"] = G.conv_net(4, (16, 16), [3, 8, 16, 8], [(5, 5), (3, 3), (3, 3)], dtype_bytes=2)
    g["reduce_kat"] = reduce_kat_graph()
    return g


REDUCE_KAT_ASSIGN = json.dumps({"k": 1, "tilings": {"x": "C", "w": "R", "z": "R"}})


def cases():
    """(name, mode, k, seed).  Corpus: acceptance.cpp:277-293 ({data, model, opt} x k in {1,2},
    seed 33) + hybrid, and test_plan.cpp:178-189 (kcuts k=2, seed 17)."""
    out = []
    corpus = ["mlp_train_d1", "mlp_train_d2", "mlp_train_d3", "mlp_train_d4", "mlp_fwd",
              "mlp_rect", "cnn_train", "cnn_fwd2"]
    for name in corpus:
        for mode in ("data", "model", "opt"):
            for k in (1, 2):
                out.append((name, mode, k, 33))
        out.append((name, "hybrid", 2, 33))
        out.append((name, "opt", 2, 17))
    for name in ("cfg1_mlp3x1024_b64", "cfg2r_mlp5x256_b64", "cfg5r_mlp3x512_b32", "fcr_alexnet_b32"):
        for k in (0, 1, 2, 3):
            out.append((name, "opt", k, 7))
        for k in (1, 2, 3):
            out.append((name, "data", k, 7))
    for k in (0, 1, 2):
        out.append(("cnnr_train_b16", "opt", k, 7))
    for k in (1, 2):
        out.append(("cnnr_train_b16", "data", k, 7))
    for k in (0, 1, 2):
        out.append(("alexr_conv_b4", "opt", k, 7))
    for k in (1, 2):
        out.append(("alexr_conv_b4", "data", k, 7))
    out.append(("alexr_conv_b4", "model", 2, 7))
    for mode, k in (("opt", 0), ("data", 1), ("opt", 1)):
        out.append(("wideconv_b2", mode, k, 7))
    out.append(("wideconv_bf16", "opt", 0, 7))
    for name, ks in (("cfg1_bf16", (0, 1)), ("cfg2r_bf16", (0, 2)), ("mlp_train_d2_bf16", (1, 2)),
                     ("fcr_alexnet_bf16", (1,)), ("alexr_conv_bf16", (0, 1))):
        for k in ks:
            out.append((name, "opt", k, 7))
        out.append((name, "data", max(ks[-1], 1), 7))
    out.append(("reduce_kat", "custom", 1, 5))
    return out


def file_stem(name, mode, k, seed):
    return f"{name}.{mode}.k{k}.s{seed}"


def make_case(gjson: str, name: str, mode: str, k: int, seed: int):
    m = REDUCE_KAT_ASSIGN if mode == "custom" else mode
    plan_text = ref.plan(gjson, m, k)
    P = json.loads(plan_text)
    sess = ref.Session(plan_text, seed)
    total = sum(int(np.prod([hi - lo for lo, hi in n["region"]])) for n in P["nodes"])
    arrays = {}
    if total <= SMALL:
        for n in P["nodes"]:
            arrays["node:" + n["id"]] = sess.node(n["id"])
        for t in P["graph"]["tensors"]:
            arrays["serial:" + t["id"]] = sess.serial(t["id"])
    else:
        for hs in P["holders"].values():
            for h in hs:
                arrays["summary:" + h] = summary(sess.node(h))
    sess.close()
    return plan_text, arrays


def main():
    check = "--check" in sys.argv
    if not ref.build():
        sys.exit("oracle/_ref is not built and /root/reference is absent")
    gs = graphs()
    os.makedirs(GOLDEN, exist_ok=True)
    bad = 0
    only = sys.argv[sys.argv.index("--only") + 1].split(",") if "--only" in sys.argv else None
    for name, mode, k, seed in cases():
        if only and name not in only:
            continue
        stem = os.path.join(GOLDEN, file_stem(name, mode, k, seed))
        plan_text, arrays = make_case(gs[name], name, mode, k, seed)
        if check:
            old = json.loads(gzip.open(stem + ".plan.json.gz", "rt").read())
            z = np.load(stem + ".values.npz")
            same = old == json.loads(plan_text) and set(z.keys()) == set(arrays) and all(
                np.array_equal(z[key], arrays[key]) for key in arrays)
            bad += not same
            print(("ok  " if same else "DIFF"), os.path.basename(stem))
            continue
        with gzip.GzipFile(stem + ".plan.json.gz", "wb", mtime=0) as f:
            f.write(plan_text.encode())
        buf = io.BytesIO()
        np.savez_compressed(buf, **arrays)
        with open(stem + ".values.npz", "wb") as f:
            f.write(buf.getvalue())
        print("wrote", os.path.basename(stem))
    if bad:
        sys.exit(f"{bad} fixtures differ from the reference")


if __name__ == "__main__":
    main()
