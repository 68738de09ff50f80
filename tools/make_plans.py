"""Emits the execution plans the benchmark runs, through the reference planner's own API
(unchanged, host C++, compiled from /root/reference by oracle/Makefile):
    graph  gen_mlp                              proj/src/graph.cpp:179-229
    plan   kcuts (opt) / preset_assignment(data) proj/src/kcuts.cpp:35-60, assign.cpp:36-81
           -> place_k(flat NVSwitch level, fanout 2^k, 9e11 B/s) -> build_execution_graph
           -> export_plan                         proj/src/execgraph.cpp:295-361
The plan document is the executor's input boundary; the planner runs offline
in the build container and the documents are committed under plans/ (gzip), so the GPU box
and the product path never load the planner.

    python tools/make_plans.py [config ...]
"""
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "plans")

# BASELINE.json configs (SURVEY §8(d) "Synthetic inputs").  All graphs are one SGD train step:
# forward, backward, update (gen_mlp backward + update), fp32 (dtype_bytes 4).
CONFIGS = {
    "cfg1_mlp3x1024_b64": (64, [1024] * 4),          # configs[0]
    "cfg2_mlp5x8192_b512": (512, [8192] * 6),        # configs[1]: 5 FC layers, hidden 8192
    "alexfc_b128": (128, [9216, 4096, 4096, 1000]),   # configs[2] FC6-FC8 component
    "vggfc_b64": (64, [25088, 4096, 4096, 1000]),     # configs[3] FC component
    "cfg5_mlp3x32768_b32": (32, [32768] * 4),        # configs[4] wide-FC stress
}
# Bounded CPU samples of each config for the reference's CPU executor (bench.py cpu_baseline
# and --impl reference): one sample through one layer (fwd, act, seed, bwd_w, bwd_x, step,
# upd) of the same width; a full sample is layers x this.
SAMPLES = {
    "cfg1_mlp3x1024_b64": ("cfg1_layer_sample_b1", 1, [1024, 1024], 3),
    "cfg2_mlp5x8192_b512": ("cfg2_layer_sample_b1", 1, [8192, 8192], 5),
    "alexfc_b128": ("alexfc_layer_sample_b1", 1, [4096, 4096], 3),
    "vggfc_b64": ("vggfc_layer_sample_b1", 1, [4096, 4096], 3),
    "cfg5_mlp3x32768_b32": ("cfg5_layer_sample_b1", 1, [32768, 32768], 3),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    names = sys.argv[1:] or list(CONFIGS)
    for name in names:
        batch, dims = CONFIGS[name]
        g = ref.gen_mlp(batch, dims)
        for mode in ("opt", "data"):
            for k in range(4):
                text = ref.plan(g, mode, k)
                P = json.loads(text)
                path = os.path.join(OUT, f"{name}.{mode}.k{k}.plan.json.gz")
                with gzip.GzipFile(path, "wb", mtime=0) as f:
                    f.write(text.encode())
                print(f"{os.path.basename(path)}: {len(P['nodes'])} nodes, "
                      f"fetch_bytes_total {P['fetch_bytes_total']}")
        sname, sb, sdims, _ = SAMPLES[name]
        text = ref.plan(ref.gen_mlp(sb, sdims), "opt", 0)
        with gzip.GzipFile(os.path.join(OUT, f"{sname}.opt.k0.plan.json.gz"), "wb", mtime=0) as f:
            f.write(text.encode())


if __name__ == "__main__":
    main()
