"""Collect the GPU parity results a test run wrote under gpurun_out/ into one committed summary,
profiles/r2_parity_fullsize.json (bench.py reports it as "parity"; it is not recomputed there):
    python tools/parity_summary.py
Sources: tests/test_gpu_parity.py (golden plans: per-op / chained worst per precision),
tests/test_gpu_fullsize.py (benched sizes: per-op, chained, every node), tests/test_gpu_peer.py
(two ranks on one GPU)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")


def load(name):
    try:
        with open(os.path.join(G, name)) as f:
            return json.load(f)
    except FileNotFoundError:
        return None


def main():
    out = {"gates_normwise": {"per_op_3xtf32": 2e-6, "per_op_tf32": 2e-3, "per_op_bf16": 1e-2,
                              "chained_3xtf32_golden": 2e-2,
                              "chained_fullsize": "<= 2 x the plain-fp32 floor (skipped when the floor > 0.1)"}}
    g = load("parity_golden.json")
    if g:
        out["golden_plans"] = {k: {"plans": len(v), "worst": max(x[0] for x in v.values()),
                                   "worst_plan": max(v.items(), key=lambda kv: kv[1][0])[0]} for k, v in g.items()}
    po = load("fullsize_per_op.json")
    if po:
        w = {}
        for key, ops in po.items():
            errs = [x["err"] for op, x in ops.items() if isinstance(x, dict) and "err" in x]
            w[key] = max(errs) if errs else None
        out["fullsize_per_op_worst"] = w
    ch = load("fullsize_chained.json")
    if ch:
        out["fullsize_chained"] = {k: {kk: vv for kk, vv in v.items() if kk != "per_tensor"} for k, v in ch.items()}
    en = load("fullsize_every_node.json")
    if en:
        out["fullsize_every_node_worst"] = en
    for w in (2, 4):
        pr = load(f"peer_{w}_rank.json")
        if pr:
            out[f"peer_{w}_ranks_one_gpu"] = pr
    path = os.path.join(ROOT, "profiles", "r2_parity_fullsize.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(path)


if __name__ == "__main__":
    main()
