"""Generate tests/golden/ fixtures from the COMPILED REFERENCE (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref):
    python tools/make_golden.py

For every case: the reference planner's plan JSON (build_execution_graph + export_plan,
execgraph.cpp:295-361), the reference's per-op graph_cost (cost.cpp:244-253), its
execute_numeric result (simulator.cpp:55-149), and the fp64 value of every node of the
reference's tiled CPU execution (via oracle/ref_driver.cpp's session, which runs
execute_numeric's node loop through the reference's own dense.cpp kernels).

Cases mirror the reference's own test corpus (proj/tests/corpus.hpp:58-103) at the seeds its
tests use (test_plan.cpp:178-223 seeds 17 and 5, acceptance.cpp:277-293 seed 33), plus
structure-preserving reductions of the BASELINE configs.
"""
from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def corpus():
    """proj/tests/corpus.hpp:58-103."""
    out = []
    for depth in range(1, 5):
        out.append((f"mlp_train_d{depth}", ref.gen_mlp(8, [8] * (depth + 1), True, True)))
    out.append(("mlp_fwd", ref.gen_mlp(16, [8, 8, 8], False, False)))
    out.append(("mlp_rect", ref.gen_mlp(8, [8, 16, 8], True, False)))
    out.append(("cnn_train", ref.gen_cnn(8, (6, 6), [2, 4], (3, 3), True)))
    out.append(("cnn_fwd2", ref.gen_cnn(16, (8, 8), [4, 4, 8], (3, 3), False)))
    return out


def reduced_baselines():
    """BASELINE configs with the same layer structure at CPU-oracle-friendly extents."""
    return [
        ("cfg1_mlp3x1024_b64", ref.gen_mlp(64, [1024] * 4, True, True)),     # cfg1 full size
        ("cfg2r_mlp5x256_b64", ref.gen_mlp(64, [256] * 6, True, True)),      # cfg2 structure
        ("cfg5r_mlp3x512_b32", ref.gen_mlp(32, [512] * 4, True, True)),      # cfg5 structure
        ("fcr_alexnet_b32", ref.gen_mlp(32, [576, 256, 256, 64], True, True)),  # AlexNet-FC shape
        ("cnnr_train_b16", ref.gen_cnn(16, (10, 10), [4, 8, 8], (3, 3), True)),
    ]


def summary(v: np.ndarray) -> np.ndarray:
    """Size-independent fingerprint of a block: sum, sum|x|, sum x^2 and 61 elements at
    fixed flat positions (used for cases too large to store whole)."""
    flat = v.reshape(-1)
    idx = np.unique(np.linspace(0, max(flat.size - 1, 0), 61).astype(np.int64))
    head = np.array([flat.sum(), np.abs(flat).sum(), (flat * flat).sum()])
    return np.concatenate([head, flat[idx]]) if flat.size else head


def write_case(name, graph, mode, k, seed, keep_all_nodes=True):
    plan = ref.plan(graph, mode, k)
    P = json.loads(plan)
    cost = ref.graph_cost(graph, mode, k)
    num = ref.execute_numeric(plan, seed)
    sess = ref.Session(plan, seed)
    arrays = {}
    holder_ids = {h for hs in P["holders"].values() for h in hs}
    for n in P["nodes"]:
        if keep_all_nodes:
            arrays["node:" + n["id"]] = sess.node(n["id"])
        elif n["id"] in holder_ids:
            arrays["summary:" + n["id"]] = summary(sess.node(n["id"]))
    if keep_all_nodes:
        for t in P["graph"]["tensors"]:
            arrays["serial:" + t["id"]] = sess.serial(t["id"])
    sess.close()
    tag = f"{name}.{mode}.k{k}.s{seed}"
    with gzip.open(os.path.join(OUT, tag + ".plan.json.gz"), "wt") as f:
        f.write(plan)
    np.savez_compressed(os.path.join(OUT, tag + ".values.npz"), **arrays)
    meta = {"case": name, "mode": mode, "k": k, "seed": seed,
            "execute_numeric": {kk: num[kk] for kk in ("max_abs", "max_rel", "values")},
            "graph_cost": {"total_bytes": cost["total_bytes"],
                           "per_op": {r["op"]: r["bytes"] for r in cost["per_op"]},
                           "forms": {r["op"]: r["form"] for r in cost["per_op"]}},
            "fetch_bytes_total": P["fetch_bytes_total"]}
    return tag, meta


def main():
    ref.build()
    os.makedirs(OUT, exist_ok=True)
    index = {}
    for name, g in corpus():
        for k in (1, 2):
            modes = ["data", "model", "opt"] + (["hybrid"] if k >= 2 else [])
            for mode in modes:
                tag, meta = write_case(name, g, mode, k, 33)
                index[tag] = meta
        tag, meta = write_case(name, g, "opt", 2, 17)   # test_plan.cpp:178-189
        index[tag] = meta
    for name, g in reduced_baselines():
        for k in (0, 1, 2, 3):
            for mode in (["opt", "data"] if k else ["opt"]):
                if name.startswith("cnnr") and k == 3:
                    continue
                tag, meta = write_case(name, g, mode, k, 7, keep_all_nodes=False)
                index[tag] = meta
    # the reducing-form known-answer plan of test_plan.cpp:191-223 (x:C, w:R, z:R, seed 5)
    g = json.dumps({"tensors": [
        {"id": "x", "shape": [4, 4], "dtype_bytes": 4, "role": "input"},
        {"id": "w", "shape": [4, 4], "dtype_bytes": 4, "role": "weight"},
        {"id": "z", "shape": [4, 4], "dtype_bytes": 4, "role": "activation"}],
        "ops": [{"id": "mm", "kind": "matmul", "inputs": ["x", "w"], "output": "z",
                 "attrs": {"transpose_a": False, "transpose_b": False}}]})
    a = json.dumps({"k": 1, "tilings": {"x": "C", "w": "R", "z": "R"}})
    tag, meta = write_case("reduce_kat", g, a, 1, 5)
    index[tag] = meta
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print(f"wrote {len(index)} cases to {OUT}")


if __name__ == "__main__":
    main()
