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
from paper_1805_04170_b200 import graphs as G  # noqa: E402

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
# Conv components of the AlexNet-/VGG-style configs (graphs.py; the FC components are above).
CONV_CONFIGS = {
    "alexconv_b128": lambda: G.alexnet_conv(128),   # configs[2] conv component
    "vggconv_b64": lambda: G.vgg_conv(64),          # configs[3] conv component
}
# Bounded CPU samples of each config for the reference's CPU executor (bench.py cpu_baseline
# and --impl reference), as BASELINE.md §2 plans them: the same structure (layer count, filter
# sizes, FULL batch) at reduced widths, re-planned by the unchanged planner at the same k, one
# step ~0.5-1 GFLOP; samples/s are extrapolated to full size by the FLOP ratio (labelled).
# cfg1 (configs[0], the reference's own CPU-runnable case) is timed at full size.
CPU_SAMPLES = {
    "cfg1_mlp3x1024_b64": lambda: ref.gen_mlp(64, [1024] * 4),
    "cfg2_mlp5x8192_b512": lambda: ref.gen_mlp(512, [256] * 6),
    "alexfc_b128": lambda: ref.gen_mlp(128, [1152, 512, 512, 125]),
    "vggfc_b64": lambda: ref.gen_mlp(64, [3136, 512, 512, 125]),
    "cfg5_mlp3x32768_b32": lambda: ref.gen_mlp(32, [1024] * 4),
    # (channel splits need multiples of 8 at k = 3)
    "alexconv_b128": lambda: G.conv_net(128, (24, 24), [3, 8, 8, 16, 16, 8], G.ALEXNET_CONV["filters"]),
    "vggconv_b64": lambda: G.conv_net(64, (29, 29), [3] + [8] * 13, G.VGG_CONV["filters"]),
}


def write(path, text):
    with gzip.GzipFile(path, "wb", mtime=0) as f:
        f.write(text.encode())


def main():
    os.makedirs(OUT, exist_ok=True)
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    bf16 = "--bf16" in sys.argv  # dtype_bytes 2 variants: plans/<name>_bf16.<mode>.k<k>
    names = args or list(CONFIGS) + list(CONV_CONFIGS)
    for name in names:
        db = 2 if bf16 else 4
        if name in CONV_CONFIGS:
            g = CONV_CONFIGS[name]()
            if bf16:
                gj = json.loads(g)
                for t in gj["tensors"]:
                    t["dtype_bytes"] = 2
                g = json.dumps(gj, sort_keys=True)
        else:
            batch, dims = CONFIGS[name]
            g = ref.gen_mlp(batch, dims, dtype_bytes=db)
        out_name = name + ("_bf16" if bf16 else "")
        for mode in ("opt", "data"):
            for k in range(4):
                text = ref.plan(g, mode, k)
                P = json.loads(text)
                path = os.path.join(OUT, f"{out_name}.{mode}.k{k}.plan.json.gz")
                write(path, text)
                print(f"{os.path.basename(path)}: {len(P['nodes'])} nodes, "
                      f"fetch_bytes_total {P['fetch_bytes_total']}")
        if bf16:
            continue
        g = CPU_SAMPLES[name]()
        for k in range(4):
            write(os.path.join(OUT, f"{name}.cpusample.opt.k{k}.plan.json.gz"), ref.plan(g, "opt", k))


if __name__ == "__main__":
    main()
