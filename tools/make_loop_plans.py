"""Loop-consistent optimal tilings (SURVEY finding 9 / §7 H1), through the UNCHANGED planner.

The planner prices ONE step: graph inputs (w) start resident for free, so its optimum keeps w
replicated and leaves w_next partitioned; the w_next -> w conversion the next step needs is
never priced.  Unrolling two steps fixes that without touching the planner: step 1's
w<l>_next IS step 2's weight input, so kcuts prices the carry.  Step 2's sub-assignment,
mapped back onto the single-step gen_mlp graph (w<l> and w<l>_next <- tiling of s1_w<l>_next,
everything else <- s2_*), is loop-consistent (w and w_next tiled alike, so the carry is a
buffer swap), and build_execution_graph on it
moves exactly the priced bytes.

    python tools/make_loop_plans.py CONFIG K [K ...]
writes plans/<config>.loop.k<K>.plan.json.gz and plans/<config>.loop.k<K>.assignment.json;
    python tools/make_loop_plans.py CONFIG K [K ...] --bf16
writes the bf16 plans of the cached assignments (plans/<config>_bf16.loop.k<K>.plan.json.gz)
(planning takes minutes: the unrolled graph's BFS levels merge, see SURVEY finding 9).
"""
import gzip
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from tools.make_plans import CONFIGS, CONV_CONFIGS  # noqa: E402

OUT = os.path.join(ROOT, "plans")


def unroll2(graph: dict) -> dict:
    weights = {t["id"] for t in graph["tensors"] if t["id"] + "_next" in
               {u["id"] for u in graph["tensors"]}}
    tensors, ops = [], []
    for s in (1, 2):
        def name(t):
            if s == 2 and t in weights:
                return f"s1_{t}_next"
            return f"s{s}_{t}"
        for t in graph["tensors"]:
            if s == 2 and t["id"] in weights:
                continue
            u = dict(t)
            u["id"] = name(t["id"])
            tensors.append(u)
        for op in graph["ops"]:
            o = json.loads(json.dumps(op))
            o["id"] = f"s{s}_{op['id']}"
            o["inputs"] = [name(i) for i in op["inputs"]]
            o["output"] = name(op["output"])
            ops.append(o)
    return {"tensors": tensors, "ops": ops}


def loop_assignment(graph: dict, unrolled_assignment: dict) -> dict:
    tilings = unrolled_assignment["tilings"]
    out = {}
    ids = {t["id"] for t in graph["tensors"]}
    for t in ids:
        if t + "_next" in ids:
            out[t] = tilings[f"s1_{t}_next"]
        elif t.endswith("_next") and t[:-5] in ids:
            # steady state: step 2's w_next feeds step 3 exactly as step 1's fed step 2
            out[t] = tilings[f"s1_{t}"]
        else:
            out[t] = tilings[f"s2_{t}"]
    return {"k": unrolled_assignment["k"], "tilings": out}


def graph_of(name, dtype_bytes=4):
    if name in CONV_CONFIGS:
        g = json.loads(CONV_CONFIGS[name]())
        for t in g["tensors"]:
            t["dtype_bytes"] = dtype_bytes
        return g
    batch, dims = CONFIGS[name] if name in CONFIGS else (8, [8] * 4)
    return json.loads(ref.gen_mlp(batch, dims, dtype_bytes=dtype_bytes))


def write_bf16(name, k):
    """The bf16 plan of the same loop-aware tiling (the optimizer minimises elements, so the
    tilings do not depend on dtype_bytes)."""
    with open(os.path.join(OUT, f"{name}.loop.k{k}.assignment.json")) as f:
        a = json.load(f)["assignment"]
    text = ref.plan(json.dumps(graph_of(name, 2)), json.dumps(a), k)
    with gzip.GzipFile(os.path.join(OUT, f"{name}_bf16.loop.k{k}.plan.json.gz"), "wb", mtime=0) as f:
        f.write(text.encode())
    print(f"{name}_bf16 k={k}: fetch_bytes_total {json.loads(text)['fetch_bytes_total']}", flush=True)


def main():
    name = sys.argv[1]
    ks = [int(a) for a in sys.argv[2:] if not a.startswith("--")]
    if "--bf16" in sys.argv:
        for k in ks:
            write_bf16(name, k)
        return
    g = graph_of(name)
    u = unroll2(g)
    for k in ks:
        t0 = time.time()
        kc = ref.kcuts(json.dumps(u), k)
        a = loop_assignment(g, {"k": k, "tilings": kc["tilings"]})
        text = ref.plan(json.dumps(g), json.dumps(a), k)
        P = json.loads(text)
        with open(os.path.join(OUT, f"{name}.loop.k{k}.assignment.json"), "w") as f:
            json.dump({"assignment": a, "unrolled_kcuts": {kk: v for kk, v in kc.items() if kk != "tilings"},
                       "plan_seconds": time.time() - t0}, f, indent=1, sort_keys=True)
        with gzip.GzipFile(os.path.join(OUT, f"{name}.loop.k{k}.plan.json.gz"), "wb", mtime=0) as f:
            f.write(text.encode())
        print(f"{name} k={k}: fetch_bytes_total {P['fetch_bytes_total']} "
              f"({time.time() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    main()
