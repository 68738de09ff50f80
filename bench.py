"""Benchmark: samples/sec of one SGD train step (forward, backward, update) executed from the
reference planner's tiling plan on N B200s, optimal tiling vs data parallel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--precision tf32|fp32|bf16]
                    [--impl ours|reference]
N > 1 runs one process per GPU (NCCL): launched by torchrun, or, when WORLD_SIZE is unset, by
this script re-launching itself under torch.distributed.run.  Plan k = log2(N), one logical
device per GPU.  Workload (BASELINE.json configs[1]): 5 FC layers, hidden 8192, batch 512
(`gen_mlp(512, [8192]*6)`), fp32 storage, random-init (seeded_tensor) weights, synthetic
inputs; plans under plans/ were emitted offline by the unchanged reference planner
(tools/make_plans.py).

A step is one iteration of the training loop: forward, backward, SGD update, and the carry of
w_next into the next step's w (TPX_FLAG_LOOP: zero-copy when the plan tiles w and w_next alike,
the carry conversion otherwise).  Timed region: K steps, CUDA events on the executor's stream,
barrier + synchronize on both sides, max over ranks.  Weights are 1.34 GB per step (> 126 MB
L2), so no L2 flush is needed between steps.

Rank 0 prints ONE JSON line.  `value` = optimal-tiling plan; `dp` = the data-parallel plan
(preset_assignment(data)) run by the same kernels in the same process.  At N = 1 the two are
the same plan (k = 0), so `variants.tiled_one_gpu` also runs k = 1..3 tiled plans on the one
GPU (the paper's tiled-on-one-GPU experiment): optimal (+ its carry), data,
and the loop-aware optimum.
"""
from __future__ import annotations

import argparse
import gzip
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
PLANS = os.path.join(ROOT, "plans")

CONFIGS = {
    "cfg2_mlp5x8192_b512": {"batch": 512, "dims": [8192] * 6, "sample": "cfg2_layer_sample_b1"},
    "cfg1_mlp3x1024_b64": {"batch": 64, "dims": [1024] * 4, "sample": "cfg1_layer_sample_b1"},
    "alexfc_b128": {"batch": 128, "dims": [9216, 4096, 4096, 1000], "sample": "alexfc_layer_sample_b1"},
    "vggfc_b64": {"batch": 64, "dims": [25088, 4096, 4096, 1000], "sample": "vggfc_layer_sample_b1"},
    "cfg5_mlp3x32768_b32": {"batch": 32, "dims": [32768] * 4, "sample": "cfg5_layer_sample_b1"},
    "alexconv_b128": {"batch": 128, "conv": True, "sample": "alexconv_layer_sample_b1"},
    "vggconv_b64": {"batch": 64, "conv": True, "sample": "vggconv_layer_sample_b1"},
}
# Whole AlexNet-/VGG-style networks: the conv component and the FC component are planned
# separately (the IR has no flatten, SURVEY finding 7) and a train step executes both plans.
NETWORKS = {
    "alexnet_b128": ["alexconv_b128", "alexfc_b128"],   # BASELINE configs[2]
    "vgg_b64": ["vggconv_b64", "vggfc_b64"],            # BASELINE configs[3]
}
METRIC = "samples/sec per train step, optimal tiling vs data-parallel, at 1/2/4/8 B200"
SEED = 7


def load_plan(name, mode, k):
    return gzip.open(os.path.join(PLANS, f"{name}.{mode}.k{k}.plan.json.gz"), "rt").read()


def graph_flops(graph):
    """Algorithmic FLOPs of one step of `graph`: 2*M*N*K per matmul plus 2*|out|*contraction per
    convolution; elementwise ops are not counted."""
    from paper_1805_04170_b200.graphs import conv_flops
    shapes = {t["id"]: t["shape"] for t in graph["tensors"]}
    f = 0
    for op in graph["ops"]:
        if op["kind"] == "matmul":
            a = shapes[op["inputs"][0]]
            kk = a[0] if op["attrs"].get("transpose_a") else a[1]
            o = shapes[op["output"]]
            f += 2 * o[0] * o[1] * kk
    return f + conv_flops(json.dumps(graph))


def parts_of(workload):
    return NETWORKS.get(workload, [workload])


def workload_batch(workload):
    return CONFIGS[parts_of(workload)[0]]["batch"]


def workload_config(workload, k):
    """The JSON line's `config` object."""
    parts = parts_of(workload)
    c = {"workload": workload, "global_batch": workload_batch(workload), "plan": f"kcuts optimal k={k}",
         "parallelism": f"tiled{1 << k}", "l2": "inputs > L2 (weights or im2col operands > 126 MB per step); no flush"}
    if len(parts) > 1 or CONFIGS[parts[0]].get("conv"):
        c["components"] = {}
        for p in parts:
            g = json.loads(load_plan(p, "opt", 0))["graph"]
            convs = [o for o in g["ops"] if o["kind"] == "conv" and o["attrs"]["mode"] == "forward"]
            sh = {t["id"]: t["shape"] for t in g["tensors"]}
            if convs:
                c["components"][p] = {"input": sh["a0"], "filters": [sh[o["inputs"][1]] for o in convs],
                                      "stride": 1, "padding": "valid"}
            else:
                c["components"][p] = {"fc_dims": CONFIGS[p]["dims"]}
    else:
        d = CONFIGS[parts[0]]["dims"]
        c.update({"hidden": d[1], "layers": len(d) - 1})
    return c


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML every 2 ms (pynvml),
    or nvidia-smi every 50 ms where NVML is unavailable."""
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = None
        self.source = "nvml"

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((float(sm), float(mx), [n for n, b in zip(self.NAMES, bits) if r & b]))
            self._stop.wait(0.002)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                r = [x.strip() for x in out.split(",")]
                if len(r) == 6 and r[0].replace(".", "").isdigit():
                    self.rows.append((float(r[0]), float(r[1]) if r[1].replace(".", "").isdigit() else None,
                                      [n for n, v in zip(self.NAMES, r[2:]) if "Active" in v and "Not" not in v]))
            except Exception:  # noqa: BLE001
                return
            self._stop.wait(0.05)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._run_nvml(nv)
        except Exception:  # noqa: BLE001
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.005)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(10)

    def summary(self):
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.rows[0][1],
                "reasons": sorted({n for r in self.rows for n in r[2]}), "samples": len(self.rows),
                "source": self.source}


def cpu_samples(workload, k, threads):
    """The reference's CPU tiled executor (execute_numeric's node loop through the reference
    library compiled from its own sources, oracle/_ref) on each component's bounded sample
    (BASELINE.md §2): the same structure -- layer count, filter sizes, FULL batch -- at reduced
    widths, planned by the unchanged planner at the same k (plans/<c>.cpusample.*,
    tools/make_plans.py).  Returns [(component, pool, FLOP ratio full : sample)]."""
    from oracle import ref
    out = []
    for p in parts_of(workload):
        text = load_plan(p + ".cpusample", "opt", k)
        full = graph_flops(json.loads(load_plan(p, "opt", 0))["graph"])
        ratio = full / graph_flops(json.loads(text)["graph"])
        out.append((p, ref.Pool(text, SEED, threads), ratio))
    return out


def cpu_rate(pools, runs, copies):
    """samples/s of the full workload: per run, each component's sample step (all copies
    concurrently) scaled by its FLOP ratio; the workload's batch per summed extrapolated time."""
    per = []
    for _ in range(runs):
        per.append(sum(pool.step() * ratio for _, pool, ratio in pools))
    return copies * len(per) / sum(per), per


def cpu_sample_text(workload, pools, copies, extra=""):
    return (f"{copies} concurrent cop{'y' if copies == 1 else 'ies'} of the reference's tiled node loop "
            f"(execute_numeric semantics, oracle/_ref built from the reference's sources, fp64, "
            f"single-threaded each) on reduced-extent graphs of the same structure at full batch "
            f"({', '.join(f'{p}: FLOP ratio full/sample {r:.4g}' for p, _, r in pools)}); samples/s "
            f"EXTRAPOLATED to full size by the FLOP ratio (the narrow samples run faster per FLOP than "
            f"the full widths: cache-resident operands, so the extrapolation favours the reference)" + extra)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import psutil
    cores = os.cpu_count() or 1
    k = int(round(math.log2(max(args.gpus, 1))))
    threads = max(1, min(cores, int(psutil.virtual_memory().available * 0.5 // (2 << 30)), 128))
    pools = cpu_samples(args.config, k, threads)
    for _, pool, _ in pools:  # one untimed pass warms caches / the allocator
        pool.step()
    v, per = cpu_rate(pools, max(1, args.steps), threads)
    v *= workload_batch(args.config)
    for _, pool, _ in pools:
        pool.close()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args.config, k),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": "reference",
                         "sample": cpu_sample_text(args.config, pools, threads,
                                                   f"; {len(per)} steps, each one sample step per copy")},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def kernel_rooflines(r, tensor_peak, hbm_peak):
    """Per GEMM class (fwd / bwd_x / bwd_w: the op id without its layer number) of this rank's
    lowered step: launches per step, mean device ms per launch (CUDA events around every lowered
    step, on the executor's stream), algorithmic FLOPs and bytes per launch (operands read once,
    every fused output written once, describe()), the bound (the larger of FLOPs / tensor peak
    and bytes / HBM peak) and the achieved rate in that unit.  Returns (list, dominant class)."""
    import re
    total = sum(r["step_ms"]) or 1.0
    cls = {}
    for st, ms in zip(r["steps_desc"], r["step_ms"]):
        if st["kind"] != "gemm":
            continue
        name = (st["part"] + ":" if st.get("part") else "") + re.sub(r"\d+$", "", st["op"])
        c = cls.setdefault(name, {"class": name, "launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0,
                                  "what": f"{'T' if st['ta'] else 'N'}{'T' if st['tb'] else 'N'} "
                                          f"{'x'.join(str(v) for v in st['shapes'][0][:3])}, "
                                          f"{st['shapes'][0][3]} fused epilogue stages, "
                                          f"{'CTA pair' if st.get('pair') else '1 CTA'}"})
        c["launches"] += 1
        c["ms"] += ms
        c["flops"] += st.get("flops", 0.0)
        c["bytes"] += st.get("min_bytes", 0.0)
    out = []
    for c in cls.values():
        n = c["launches"]
        t_tc = c["flops"] / (tensor_peak * 1e12)
        t_hbm = c["bytes"] / (hbm_peak * 1e9)
        bound = "tensor" if t_tc >= t_hbm else "hbm"
        sec = c["ms"] / 1e3
        ach = c["flops"] / sec / 1e12 if bound == "tensor" else c["bytes"] / sec / 1e9
        pk = tensor_peak if bound == "tensor" else hbm_peak
        out.append({"class": c["class"], "what": c["what"], "launches_per_step": n, "ms": c["ms"] / n,
                    "share": c["ms"] / total, "bound": bound, "unit": "TFLOP/s" if bound == "tensor" else "GB/s",
                    "achieved": ach, "peak": pk, "frac": ach / pk,
                    "per_launch": {"flops": c["flops"] / n, "bytes": c["bytes"] / n},
                    "tflops": c["flops"] / sec / 1e12, "gbs": c["bytes"] / sec / 1e9,
                    "roofline_ms": max(t_tc, t_hbm) * 1e3 / n})
    out.sort(key=lambda c: -c["share"])
    return out, (out[0] if out else None)


def step_roofline_ms(kernels):
    return sum(k["roofline_ms"] * k["launches_per_step"] for k in kernels)


def measured_traffic():
    """DRAM bytes per launch of each GEMM class from the committed ncu --set full capture
    (profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


def timed_once(fn, stream, barrier):
    """Device time of fn() (which enqueues its own steps) on `stream`, CUDA events, barriers."""
    import torch
    barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    barrier()
    return a.elapsed_time(b)


def timed(fn, stream, steps, barrier):
    import torch
    barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    barrier()
    return a.elapsed_time(b)


def relaunch(args):
    """--gpus N > 1 without a torchrun environment: one process per GPU through
    torch.distributed.run on this node (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def plan_exists(name, mode, k):
    return os.path.exists(os.path.join(PLANS, f"{name}.{mode}.k{k}.plan.json.gz"))


def parity_summary():
    """The committed full-size parity results this code was gated by (tests/test_gpu_fullsize.py
    writes them; profiles/ holds the copy from the last GPU run): reported, not recomputed."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_parity_fullsize.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2_mlp5x8192_b512", choices=sorted(CONFIGS) + sorted(NETWORKS))
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32", "bf16"])
    ap.add_argument("--no-variants", action="store_true", help="skip the bf16 / fp32 / tiled variants")
    ap.add_argument("--no-graph", action="store_true", help="launch the lowered steps one by one")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--xchg", default="peer", choices=["peer", "nccl"],
                    help="N > 1 cross-rank fetches: peer pulls over NVLink (CUDA IPC) or NCCL send/recv")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch(args))  # one process per GPU (both arms launch the same way)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_1805_04170_b200.executor import (FLAG_FORCE_XCHG, FLAG_FUSE, FLAG_GRAPH, FLAG_LOOP, FLAG_PEER,
                                                FLAG_PEER_SOLO, Context, PlanExecutor)
    for kv in filter(None, os.environ.get("TPX_GEMM_KNOBS", "").split(",")):  # development A/B only
        import ctypes
        from paper_1805_04170_b200 import native
        kk, vv = kv.split(":")
        native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(int(kk)), ctypes.c_uint(int(vv)))

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    k = int(round(math.log2(world)))
    if 1 << k != world or k > 3:
        raise SystemExit("N must be 1, 2, 4 or 8")
    # TPX_BENCH_SHARE_GPU=1: every rank on cuda:0 (exercises the N > 1 code path -- peer pulls
    # between processes, counters, barriers -- on a one-GPU box; its numbers are not scaling data)
    share = os.environ.get("TPX_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if torch.cuda.device_count() < world and world > 1 and local >= torch.cuda.device_count():
        raise SystemExit(f"--gpus {world} needs {world} GPUs; this node has {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    peer = world > 1 and args.xchg == "peer"
    if world > 1:
        # peer mode moves no data through torch.distributed (only IPC handles, barriers and the
        # max over ranks of the device times), so gloo suffices; NCCL mode needs the NCCL group
        if peer:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if peer else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    parts = parts_of(args.config)
    batch = workload_batch(args.config)
    prec = 1 if args.precision == "fp32" else 0  # bf16: storage type comes from the bf16 plan
    ctx = Context(local, rank, world)
    if world > 1 and (not peer or not share):
        # NCCL mode exchanges through this communicator; peer mode pulls over CUDA IPC and keeps
        # it only as the stand-by route (ranks sharing one GPU cannot form one)
        try:
            ctx.init_comm_from_torch()
            print(f"[bench] rank {rank}: NCCL communicator initialised (nranks={world}, device cuda:{local})"
                  + (" -- data path: peer pulls over NVLink (CUDA IPC)" if peer else ""), file=sys.stderr, flush=True)
        except Exception as e:  # noqa: BLE001
            if not peer:
                raise
            print(f"[bench] rank {rank}: no NCCL communicator ({e}); peer mode does not need one",
                  file=sys.stderr, flush=True)
    stream = torch.cuda.Stream()
    hbm_peak, bf16_peak, peak_kind = peaks()
    base_flags = FLAG_FUSE | FLAG_LOOP | (0 if args.no_graph else FLAG_GRAPH) | (FLAG_PEER if peer else 0)
    announced = []

    def load(mode, suffix, kk, prec, flags):
        exs, texts = [], []
        for part in parts:
            text = load_plan(part + suffix, mode, kk)
            ex = PlanExecutor(ctx, text, precision=prec, flags=flags)
            if (flags & FLAG_PEER) and world > 1:
                ex.connect_peers_from_torch()  # every rank maps every other rank's arena (CUDA IPC)
                if not announced:
                    announced.append(1)
                    print(f"[bench] rank {rank}: peer arenas of {world} ranks mapped over NVLink (CUDA IPC), "
                          f"device cuda:{local}", file=sys.stderr, flush=True)
            ex.set_stream(stream.cuda_stream)
            ex.init_inputs(SEED)
            exs.append(ex)
            texts.append(text)
        return exs, texts

    def stats_of(exs):
        sts = [ex.stats() for ex in exs]
        st = {key: sum(x[key] for x in sts) for key in sts[0]}
        d = [ex.describe() for ex in exs]
        st["carry_bytes"] = sum(x["carry_bytes"] for x in d)
        st["carry_launches"] = sum(len(x["carry"]["steps"]) for x in d)
        st["swapped"] = sum(len(x["swapped"]) for x in d)
        return st

    def conversion_times(exs):
        """Time-model parity: the planner's time model prices a phase at its
        bytes over the link bandwidth (simulate_traffic, proj/src/simulator.cpp:40-47).  Here the
        link of a one-GPU tiled run is HBM (a fetch reads and writes its bytes once), so the model
        is est = sum over phases of 2 x bytes / HBM peak; measured = the device time of the
        lowered conversion steps (copies / pulls / reductions / syncs; CUDA events per step,
        graph replay off), median of 3 steps."""
        conv = ("copy", "pull", "pack", "nccl", "reduce", "signal", "barrier")
        runs = []
        for _ in range(3):
            t = 0.0
            for ex in exs:
                ex.enable_timing(True)
                ex.execute()
                steps = ex.describe()["main"]["steps"]
                t += sum(ms for ms, st in zip(ex.last_step_times(), steps) if st.get("what") in conv)
                ex.enable_timing(False)
            runs.append(t)
        est = sum(2.0 * v for ex in exs for v in ex.describe()["per_phase_fetch_bytes_in"].values()) / (hbm_peak * 1e9)
        meas = statistics.median(runs) / 1e3
        return {"est_seconds_hbm": est, "measured_conversion_seconds": meas,
                "measured_over_model": meas / est if est else None}

    def quick(mode, suffix, kk, prec, flags, steps, model=False):
        """A plan set timed alone (variants): warm-up, then `steps` loop steps."""
        exs, _ = load(mode, suffix, kk, prec, flags)
        try:
            def step():
                for ex in exs:
                    ex.execute()
            for _ in range(args.warmup):
                step()
            ms = max_over_ranks(timed(step, stream, steps, barrier))
            st = stats_of(exs)
            tm = conversion_times(exs) if model and st["fetch_bytes_total"] else None
        finally:
            for ex in exs:
                ex.close()
        r = {"value": batch * steps / (ms / 1e3), "ms_per_step": ms / steps,
             "fetch_bytes_total": st["fetch_bytes_total"], "carry_bytes_per_step": st["carry_bytes"],
             "launches_per_step": st["n_kernel_launches"] + st["carry_launches"]}
        if tm:
            r["time_model"] = tm
        return r

    def n_gpu_projection(steps):
        """One rank's share of an N-GPU step, measured on this GPU (TPX_FLAG_PEER_SOLO: the rank's
        own program -- its GEMMs on its shards, its pull launches reading local HBM instead of
        NVLink, its sync points already satisfied), for ranks 0 and N-1 of N = 2, 4, 8.  The
        projection adds the rank's pulled bytes at NVLink 5 bandwidth (900 GB/s per direction)
        without overlap: projected step = max over the two ranks of (measured + bytes / 900 GB/s).
        A projection from measured per-GPU work, not a multi-GPU measurement."""
        out = {}
        for kk in (1, 2, 3):
            row = {}
            for mode in ("loop", "opt", "data"):
                if not all(plan_exists(p + suffix, mode, kk) for p in parts):
                    continue
                per_rank = []
                for rk in sorted({0, (1 << kk) - 1}):
                    sctx = Context(local, rk, 1 << kk)
                    exs = []
                    try:
                        for part in parts:
                            ex = PlanExecutor(sctx, load_plan(part + suffix, mode, kk), precision=prec,
                                              flags=base_flags | FLAG_PEER | FLAG_PEER_SOLO)
                            ex.set_stream(stream.cuda_stream)
                            ex.init_inputs(SEED)
                            exs.append(ex)

                        def step():
                            for ex in exs:
                                ex.execute()
                        for _ in range(args.warmup):
                            step()
                        ms = timed(step, stream, steps, barrier) / steps
                        xin = sum(ex.stats()["rank_xrank_bytes_in"] for ex in exs)
                    finally:
                        for ex in exs:
                            ex.close()
                        sctx.close()
                    per_rank.append({"rank": rk, "measured_ms": ms, "pulled_bytes": xin,
                                     "projected_ms": ms + xin / 900e9 * 1e3})
                proj = max(r["projected_ms"] for r in per_rank)
                row[mode] = {"per_rank": per_rank, "projected_ms_per_step": proj,
                             "projected_samples_per_s": batch / (proj / 1e3)}
            if "data" in row:
                for m in ("loop", "opt"):
                    if m in row:
                        row[f"{m}_vs_dp"] = row[m]["projected_samples_per_s"] / row["data"]["projected_samples_per_s"]
            out[f"N{1 << kk}"] = row
        return out

    def measure(mode, suffix, prec):
        """One plan set (every component of the workload) timed end to end."""
        exs, texts = load(mode, suffix, k, prec, base_flags)
        st = stats_of(exs)

        def step():
            for ex in exs:
                ex.execute()

        for _ in range(args.warmup):
            step()
        clk = ClockSampler(local)
        with clk:
            ms = timed(step, stream, args.steps, barrier)
        ms = max_over_ranks(ms)
        r = {"ms_per_step": ms / args.steps, "value": batch * args.steps / (ms / 1e3),
             "stats": st, "clocks": clk.summary()}
        # per-launch timing pass (events between every lowered step) for the roofline
        g_ms, t_ms, per_step, desc = [], [], [], []
        for ex, part in zip(exs, parts):
            ex.enable_timing(True)
            ex.init_inputs(SEED)  # restart the loop: the timing pass runs the first program
            desc += [dict(d, part=part if len(parts) > 1 else "") for d in ex.describe()["main"]["steps"]]
        for _ in range(5):
            g = t = 0.0
            ps = []
            for ex in exs:
                ex.init_inputs(SEED)
                ex.execute()
                tt = ex.last_timing()
                g += tt["gemm_ms"]
                t += tt["total_ms"]
                ps += ex.last_step_times()
            g_ms.append(g)
            t_ms.append(t)
            per_step.append(ps)
        for ex in exs:
            ex.enable_timing(False)
            ex.init_inputs(SEED)
        r["gemm_ms"] = statistics.median(g_ms)
        r["timed_total_ms"] = statistics.median(t_ms)
        r["step_ms"] = [statistics.median(x) for x in zip(*per_step)]
        r["steps_desc"] = desc
        # e2e through the public API: every component's graph input (x0 / a0) from pinned host
        # memory in, the component's network output (the seed op's input) out, every step.
        # The copies run on a copy stream and overlap compute the way a training loop does:
        # step i+1's batch streams in (H2D into a device staging buffer) while step i runs,
        # and step i's network output streams out (D2H) during its own backward pass, right
        # after the lowered step that produces it (tpx_execute_steps splits the step there).
        hin, hout, splits = [], [], []
        for ex, text in zip(exs, texts):
            plan = json.loads(text)
            mine = set(ex.my_devices())
            nodes = {n["id"]: n for n in plan["nodes"]}
            roles = {t["id"]: t["role"] for t in plan["graph"]["tensors"]}
            src = [t for t, rl in roles.items() if rl == "input"]
            last = next(o["inputs"][0] for o in plan["graph"]["ops"] if o["id"] == "seed")
            hdt = torch.bfloat16 if ex.storage_bytes() == 2 else torch.float32  # raw storage I/O
            for t in src:
                for h in plan["holders"][t]:
                    if nodes[h]["device"] in mine:
                        n = math.prod(ex.node_shape(h))
                        hin.append((ex, h, torch.empty(n, dtype=hdt, pin_memory=True).uniform_(-1, 1),
                                    torch.empty(n, dtype=hdt, device="cuda")))
            for h in plan["holders"][last]:
                if nodes[h]["device"] in mine:
                    n = math.prod(ex.node_shape(h))
                    hout.append((ex, h, torch.empty(n, dtype=hdt, pin_memory=True),
                                 torch.empty(n, dtype=hdt, device="cuda")))
            # first lowered step after which the output exists: the last step of its producer
            # op, or of the op it is fused into (walk the producer chain back to a step)
            ops = {o["output"]: o for o in plan["graph"]["ops"]}
            steps = ex.describe()["main"]["steps"]
            t, split = last, None
            while split is None and t in ops:
                idx = [i for i, stp in enumerate(steps) if stp["op"] == ops[t]["id"]]
                if idx:
                    split = max(idx) + 1
                else:
                    t = ops[t]["inputs"][0]
            splits.append(split if split is not None else len(steps))
        h2d = sum(v.numel() * v.element_size() for _, _, v, _ in hin)
        d2h = sum(v.numel() * v.element_size() for _, _, v, _ in hout)
        nsteps = [len(ex.describe()["main"]["steps"]) for ex in exs]
        copy = torch.cuda.Stream()
        in_ready = torch.cuda.Event()
        out_read = torch.cuda.Event()  # the previous step's D2H has read the output staging

        def stage_inputs():  # next batch: pinned host -> device staging, on the copy stream
            with torch.cuda.stream(copy):
                for _, _, hv, dv in hin:
                    dv.copy_(hv, non_blocking=True)
                in_ready.record(copy)

        def e2e_step():
            stream.wait_event(in_ready)
            for ex, h, _, dv in hin:
                ex.copy_node_device(h, dv.data_ptr(), dv.numel(), True)
            consumed = torch.cuda.Event()
            consumed.record(stream)
            copy.wait_event(consumed)
            stage_inputs()
            for ex, sp, ns in zip(exs, splits, nsteps):
                ex.execute_steps(0, sp)
                outs = [(h, hv, dv) for e2, h, hv, dv in hout if e2 is ex]
                if outs:
                    stream.wait_event(out_read)  # no overwrite of dv before its D2H has read it
                for h, _, dv in outs:
                    ex.copy_node_device(h, dv.data_ptr(), dv.numel(), False)
                if outs:
                    produced = torch.cuda.Event()
                    produced.record(stream)
                    copy.wait_event(produced)
                    with torch.cuda.stream(copy):
                        for _, hv, dv in outs:
                            hv.copy_(dv, non_blocking=True)
                    out_read.record(copy)
                ex.execute_steps(sp, ns)

        def e2e_run():
            for _ in range(args.steps):
                e2e_step()
            stream.wait_stream(copy)  # the last step's output has reached the host

        out_read.record(copy)
        stage_inputs()
        for _ in range(2):
            e2e_step()
        stream.wait_stream(copy)
        e_ms = max_over_ranks(timed_once(e2e_run, stream, barrier))
        tot = torch.tensor([h2d, d2h], dtype=torch.float64, device="cpu" if peer else "cuda")
        if world > 1:
            dist.all_reduce(tot)
        r["e2e"] = {"value": batch * args.steps / (e_ms / 1e3), "unit": "samples/s",
                    "h2d_bytes_per_step": int(tot[0].item()), "d2h_bytes_per_step": int(tot[1].item()),
                    "copies": ("every step: its inputs pinned host -> device (prefetched on a copy stream "
                               "during the previous step, then device -> plan buffers) and its network "
                               "output device -> pinned host on the copy stream during its backward "
                               "pass; the timed region ends after the last output lands on the host")}
        for ex in exs:
            ex.close()
        return r

    res = {}
    suffix = "_bf16" if args.precision == "bf16" else ""
    for mode in ("opt", "data"):
        res[mode] = measure(mode, suffix, prec)
    # N > 1: the optimal tiling of the TRAINING LOOP is the loop-consistent kcuts optimum (SURVEY
    # finding 9 / §7 H1 (a): w and w_next tiled alike, every byte priced); the planner's
    # single-step optimum (+ its unpriced w_next -> w carry) is reported beside it
    if k >= 1 and all(plan_exists(p + suffix, "loop", k) for p in parts):
        res["loop"] = measure("loop", suffix, prec)
    variants = {}
    if not args.no_variants:
        vsteps = max(5, min(args.steps, 20))
        # the other storage / arithmetic modes of the same plan
        others = [("bf16", "_bf16", 0)] if args.precision != "bf16" else []
        if args.precision != "fp32":
            others.append(("fp32_3xtf32", "", 1))
        for name, sfx, pv in others:
            if all(plan_exists(p + sfx, "opt", k) for p in parts):
                variants[name] = dict(quick("opt", sfx, k, pv, base_flags, vsteps),
                                      plan=f"kcuts optimal k={k}" + (", graph dtype_bytes 2" if sfx else ""))
        if world == 1:
            # tiled on one GPU: 2^kk logical devices share the GPU, fetches are HBM copies
            free = torch.cuda.mem_get_info()[0]
            tiled = {}
            for kk in (1, 2, 3):
                row = {}
                for label, mode, flags in (("opt", "opt", base_flags), ("opt_step_only", "opt", base_flags & ~FLAG_LOOP),
                                           ("data", "data", base_flags), ("loop", "loop", base_flags),
                                           ("loop_peer_path", "loop", base_flags | FLAG_FORCE_XCHG | FLAG_PEER)):
                    if not all(plan_exists(p + suffix, mode, kk) for p in parts):
                        continue
                    probe = [PlanExecutor(Context.host_only(), load_plan(p + suffix, mode, kk)) for p in parts]
                    need = sum(x.stats()["device_bytes"] for x in probe)
                    if need > 0.85 * free:
                        row[label] = {"skipped": f"arena {need / 2**30:.1f} GiB > 85% of free HBM"}
                        continue
                    row[label] = quick(mode, suffix, kk, prec, flags, vsteps, model=label in ("opt_step_only", "data"))
                if "data" in row and "value" in row["data"]:
                    for lab in ("opt", "opt_step_only", "loop", "loop_peer_path"):
                        if "value" in row.get(lab, {}):
                            row[f"{lab}_vs_dp"] = row[lab]["value"] / row["data"]["value"]
                tiled[f"k{kk}"] = row
            variants["tiled_one_gpu"] = tiled
            variants["n_gpu_projection"] = n_gpu_projection(vsteps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            pools = cpu_samples(args.config, 0, 1)
            for _, pool, _ in pools:
                pool.step()
            v, per = cpu_rate(pools, 3, 1)
            for _, pool, _ in pools:
                pool.close()
            cpu = {"value": v * batch, "unit": "samples/s", "cores": 1, "kind": "reference",
                   "sample": cpu_sample_text(args.config, pools, 1,
                                             f"; 3 runs after 1 warm-up, {sum(per):.1f} s extrapolated")}
            if args.config != "cfg1_mlp3x1024_b64":
                # configs[0], the reference's own CPU-runnable case, at FULL size in the same run
                from oracle import ref
                pool = ref.Pool(load_plan("cfg1_mlp3x1024_b64", "opt", 0), SEED, 1)
                t = pool.step()
                pool.close()
                cpu["cfg1_full_size"] = {"value": 64 / t, "unit": "samples/s", "seconds_per_step": t,
                                         "sample": "cfg1 (gen_mlp(64, [1024]*4)) full train step, k=0 plan"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "samples/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    xin = max_over_ranks(float(res.get("loop", res["opt"])["stats"]["rank_xrank_bytes_in"]))
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    d = res["data"]
    o = res.get("loop", res["opt"])
    single = res["opt"]
    flops = o["stats"]["gemm_flops"]
    # north_star step roofline per GPU: max(FLOPs at the tensor peak, received bytes at NVLink
    # bandwidth); the HBM term of the GEMMs is reported beside it
    nvl_bw = 900e9  # NVLink 5 per direction per GPU (B200 datasheet; not measurable on one GPU)
    tf32_peak = bf16_peak / 2
    peak = bf16_peak if args.precision == "bf16" else tf32_peak if prec == 0 else tf32_peak / 3
    kernels, dom = kernel_rooflines(o, peak, hbm_peak)
    traffic = (measured_traffic().get(dom["class"]) or {}).get("dram_bytes_per_launch") if dom else None
    line = {
        "metric": METRIC, "value": o["value"], "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": o["ms_per_step"],
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": {"tf32": "tf32", "fp32": "fp32(3xtf32)", "bf16": "bf16"}[args.precision],
        "data": "synthetic",
        "config": dict(workload_config(args.config, k),
                       plan=(f"loop-consistent kcuts optimum k={k} (unrolled-2-step planning through the unchanged "
                             f"planner API, SURVEY finding 9)" if "loop" in res else f"kcuts optimal k={k}"),
                       exchange=("peer pull over NVLink (CUDA IPC), device-side phase counters" if peer else
                                 "NCCL send/recv per phase" if world > 1 else "one rank: HBM copies")),
        "dp": {"value": d["value"], "ms_per_step": d["ms_per_step"], "plan": f"preset data k={k}",
               "e2e": d["e2e"]["value"], "fetch_bytes_total": d["stats"]["fetch_bytes_total"],
               "carry_bytes_per_step": d["stats"]["carry_bytes"]},
        "opt_vs_dp": o["value"] / d["value"],
        "opt_single_step": ({"value": single["value"], "ms_per_step": single["ms_per_step"],
                             "plan": f"kcuts single-step optimum k={k} + its w_next -> w carry (unpriced by the planner)",
                             "carry_bytes_per_step": single["stats"]["carry_bytes"],
                             "vs_dp": single["value"] / d["value"]} if "loop" in res else None),
        "fetch_bytes_total": o["stats"]["fetch_bytes_total"],
        "carry_bytes_per_step": o["stats"]["carry_bytes"],
        "loop_carry": (f"{o['stats']['swapped']} weights carried by buffer swap (zero copy), "
                       f"{o['stats']['carry_bytes']} cross-device bytes of w_next -> w conversion per step "
                       f"(unpriced by the planner) in {o['stats']['carry_launches']} extra launches"),
        "e2e": o["e2e"],
        "gpu_launches": int((o["stats"]["n_kernel_launches"] + o["stats"]["carry_launches"]) * args.steps),
        "roofline": {"bound": dom["bound"], "kernel": f"tcgen05 tile GEMM, {dom['class']} ({dom['what']})",
                     "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                     "frac": dom["achieved"] / dom["peak"], "traffic": traffic,
                     "algorithmic_per_launch": dom["per_launch"], "avg_launch_ms": dom["ms"],
                     "share_of_step": dom["share"],
                     "peak_basis": (f"{peak_kind} MEASURED_PEAKS: HBM {hbm_peak} GB/s; tensor = bf16 {bf16_peak} "
                                    f"TFLOP/s" + ("" if args.precision == "bf16" else
                                                  " / 2 (kind::tf32 issues at half the kind::f16 rate)")
                                    + (" / 3 (3xTF32 split)" if prec else "")),
                     "kernels": kernels,
                     "flops_per_step": flops, "gemm_ms_per_step": o["gemm_ms"],
                     "gemm_share_of_step": o["gemm_ms"] / o["timed_total_ms"],
                     "timing_pass": ("per-launch CUDA events between every lowered step, graph replay off; "
                                     "shares are of that pass's total"),
                     "step_roofline_ms": step_roofline_ms(kernels),
                     "step_frac": step_roofline_ms(kernels) / o["ms_per_step"],
                     "north_star_step": {
                         "tensor_ms": flops / (peak * 1e12) * 1e3,
                         "nvlink_ms": xin / nvl_bw * 1e3,
                         "hbm_gemm_ms": step_roofline_ms(kernels),
                         "roofline_ms": max(flops / (peak * 1e12) * 1e3, xin / nvl_bw * 1e3),
                         "frac": max(flops / (peak * 1e12) * 1e3, xin / nvl_bw * 1e3) / o["ms_per_step"],
                         "frac_3term": max(flops / (peak * 1e12) * 1e3, xin / nvl_bw * 1e3,
                                           step_roofline_ms(kernels)) / o["ms_per_step"],
                         "received_bytes_per_gpu": xin,
                         "basis": "per GPU: this rank's GEMM FLOPs at the measured tensor peak; the most bytes any "
                                  "rank pulls from other ranks at 900 GB/s NVLink; hbm_gemm_ms = sum over GEMM "
                                  "launches of max(FLOPs/tensor peak, bytes/HBM peak)"}},
        "clocks": o["clocks"],
        "cpu_baseline": cpu,
        "variants": variants,
        "parity": parity_summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
