"""Host-side mirror of the reference's plan-execution interface, over the C ABI (tpx.h).

Reference interface (proj/include/tileplan/simulator.hpp:36-45):
    struct NumericCheck { double max_abs, max_rel; int64_t values; uint64_t seed; };
    NumericCheck execute_numeric(const ExecutionPlan& p, uint64_t seed);
Here `execute_numeric(plan_json, seed)` runs the plan's per-device nodes on the GPU through the
native executor and checks every holder block of every tensor against a single-device run of
the same graph on the same GPU (the B200 counterpart of serial_execute,
proj/src/oracle.cpp:176-202: the graph lowered as a one-device plan, every op one sub-op),
with the same metric: max |d| and max |d| / max(|serial|, 1) (simulator.cpp:129-147).

Errors from the native side raise `TpxError` carrying the library's message, the analogue of
tileplan::Error.  No CPU compute path exists: without the CUDA library every call raises.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

from . import native
from .native import TpxError, check, lib

PREC_TF32 = 0
PREC_FP32 = 1
FLAG_FUSE = 1
FLAG_FORCE_XCHG = 2
FLAG_DIRECT_CONV = 4  # convolutions as direct CUDA-core loops (cross-check of the tcgen05 lowering)
FLAG_GRAPH = 8        # the whole step replayed as one CUDA graph
FLAG_LOOP = 16        # execute() = one training-loop step: the weights carry into the next step
FLAG_PEER = 32        # cross-rank fetches pulled from the peers' arenas over NVLink (CUDA IPC)
FLAG_KMAJOR_CONV = 64  # conv grad_input on transposed K-major operands (opt-in)
FLAG_PEER_SOLO = 128  # one rank of an N-rank peer plan alone on this GPU (timing projection only)


@dataclass
class NumericCheck:
    max_abs: float = 0.0
    max_rel: float = 0.0
    values: int = 0
    seed: int = 0


class Context:
    """One process's share of the job: a CUDA device (or host-only) and its rank."""

    def __init__(self, cuda_ordinal: int = 0, rank: int = 0, world: int = 1):
        h = ctypes.c_void_p()
        check(lib().tpx_create(cuda_ordinal, rank, world, ctypes.byref(h)))
        self._h = h
        self.rank, self.world, self.ordinal = rank, world, cuda_ordinal

    @classmethod
    def host_only(cls, rank: int = 0, world: int = 1) -> "Context":
        return cls(-1, rank, world)

    def init_comm_from_torch(self):
        """Create the NCCL communicator; the 128-byte unique id travels over the default
        torch.distributed group (plumbing only)."""
        import torch
        import torch.distributed as dist

        buf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            check(lib().tpx_comm_unique_id(buf, 128))
        t = torch.tensor(list(buf.raw), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0)
        raw = bytes(t.cpu().tolist())
        check(lib().tpx_init_comm(self._h, raw, 128))

    def close(self):
        if getattr(self, "_h", None):
            lib().tpx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PlanExecutor:
    """A loaded, lowered plan on one rank."""

    def __init__(self, ctx: Context, plan_json: str, precision: int = PREC_TF32,
                 flags: int = FLAG_FUSE):
        self.ctx = ctx
        self.plan_text = plan_json if isinstance(plan_json, str) else plan_json.decode()
        raw = self.plan_text.encode()
        h = ctypes.c_void_p()
        check(lib().tpx_load_plan(ctx._h, raw, len(raw), precision, flags, ctypes.byref(h)))
        self._h = h
        self.plan = json.loads(self.plan_text)
        self._nodes = {n["id"]: n for n in self.plan["nodes"]}

    # ---------------------------------------------------------------- peer mode
    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        check(lib().tpx_plan_ipc_handle(self._h, buf, 64))
        return buf.raw

    def connect_peers(self, handles: List[bytes]):
        raw = b"".join(handles)
        check(lib().tpx_plan_connect_peers(self._h, raw, len(raw)))

    def connect_peers_from_torch(self, group=None):
        """FLAG_PEER with world > 1: all-gather the arenas' 64-byte CUDA IPC handles over the
        torch.distributed group (plumbing only) and map the peers' arenas."""
        import torch.distributed as dist
        handles = [None] * self.ctx.world
        dist.all_gather_object(handles, self.ipc_handle(), group=group)
        self.connect_peers(handles)

    # ---------------------------------------------------------------- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().tpx_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- execution
    def set_stream(self, stream_handle: int):
        check(lib().tpx_set_stream(self._h, int(stream_handle)))

    def init_inputs(self, seed: int):
        check(lib().tpx_init_inputs(self._h, seed))

    def execute(self):
        check(lib().tpx_execute(self._h))

    def execute_op(self, op_id: str):
        check(lib().tpx_execute_op(self._h, op_id.encode()))

    def carry_weights(self):
        check(lib().tpx_carry_weights(self._h))

    def synchronize(self):
        check(lib().tpx_synchronize(self._h))

    def enable_timing(self, on: bool = True):
        check(lib().tpx_enable_timing(self._h, int(on)))

    def last_step_times(self):
        """Per lowered step device ms of the last timed execute() (describe()['main']['steps'] order)."""
        n = ctypes.c_int64()
        check(lib().tpx_last_step_times(self._h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_double * max(n.value, 1))()
        check(lib().tpx_last_step_times(self._h, buf, n.value, ctypes.byref(n)))
        return list(buf[: n.value])

    def last_timing(self):
        t, g, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        check(lib().tpx_last_timing(self._h, ctypes.byref(t), ctypes.byref(g), ctypes.byref(c)))
        return {"total_ms": t.value, "gemm_ms": g.value, "copy_ms": c.value}

    # ---------------------------------------------------------------- node values
    def node_shape(self, node_id: str):
        if node_id not in self._nodes:
            raise TpxError(f"unknown node '{node_id}'")
        return [hi - lo for lo, hi in self._nodes[node_id]["region"]]

    def read_node(self, node_id: str) -> np.ndarray:
        shape = self.node_shape(node_id)
        out = np.empty(shape, dtype=np.float64)
        check(lib().tpx_read_node(self._h, node_id.encode(),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.size))
        return out

    def write_node(self, node_id: str, value: np.ndarray):
        v = np.ascontiguousarray(value, dtype=np.float64)
        if list(v.shape) != self.node_shape(node_id):
            raise TpxError(f"value for node {node_id} has shape {list(v.shape)}, "
                           f"node region is {self.node_shape(node_id)}")
        check(lib().tpx_write_node(self._h, node_id.encode(),
                                   v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), v.size))

    # Raw storage I/O: n elements of the plan's storage type (fp32, or bf16 for dtype_bytes-2
    # plans; see storage_bytes()) between host memory and a node's holder block.
    def read_node_f32_into(self, node_id: str, host_ptr: int, n: int):
        check(lib().tpx_read_node_f32(self._h, node_id.encode(), ctypes.c_void_p(host_ptr), n))

    def write_node_f32_from(self, node_id: str, host_ptr: int, n: int):
        check(lib().tpx_write_node_f32(self._h, node_id.encode(), ctypes.c_void_p(host_ptr), n))

    def execute_steps(self, begin: int, end: int):
        """Lowered steps [begin, end) (describe()['main']['steps'] order) on the plan stream."""
        check(lib().tpx_execute_steps(self._h, int(begin), int(end)))

    def copy_node_device(self, node_id: str, dev_ptr: int, n: int, to_node: bool):
        """Device-to-device copy between a node and n contiguous storage elements at dev_ptr."""
        check(lib().tpx_copy_node_device(self._h, node_id.encode(), ctypes.c_void_p(dev_ptr), n, int(to_node)))

    def storage_bytes(self) -> int:
        return int(self.stats()["storage_bytes"])

    def node_view(self, node_id: str):
        p, r = ctypes.c_uint64(), ctypes.c_int()
        sh, st = (ctypes.c_int64 * 4)(), (ctypes.c_int64 * 4)()
        check(lib().tpx_node_view(self._h, node_id.encode(), ctypes.byref(p), ctypes.byref(r), sh, st))
        return p.value, list(sh)[: r.value], list(st)[: r.value]

    def holders(self) -> Dict[str, List[str]]:
        return self.plan["holders"]

    def my_devices(self) -> List[int]:
        n, w, r = self.plan.get("devices", 1 << self.plan["k"]), self.ctx.world, self.ctx.rank
        return [d for d in range(n) if (d * w) // n == r]

    # ---------------------------------------------------------------- accounting
    def stats(self) -> dict:
        s = native.Stats()
        check(lib().tpx_plan_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def describe(self) -> dict:
        p = ctypes.c_void_p()
        check(lib().tpx_plan_describe(self._h, ctypes.byref(p)))
        try:
            return json.loads(ctypes.string_at(p).decode())
        finally:
            lib().tpx_free_string(p)


def serial_plan(graph: dict) -> str:
    """The graph as a one-device plan (what build_execution_graph emits for k = 0,
    execgraph.cpp:190-290): a buffer node per graph input, one sub_op per op, holders = the
    sub_ops / buffers.  Executing it is the device-side serial_execute."""
    nodes, holders, holder_of = [], {}, {}
    produced = {op["output"] for op in graph["ops"]}
    shapes = {t["id"]: t["shape"] for t in graph["tensors"]}
    cnt = 0

    def add(n):
        nonlocal cnt
        n["id"] = f"n{cnt}"
        cnt += 1
        nodes.append(n)
        return n["id"]

    for t in sorted(shapes):
        if t in produced:
            continue
        holder_of[t] = add({"kind": "buffer", "device": 0, "tensor": t, "phase": "init",
                            "region": [[0, e] for e in shapes[t]]})
    for op in graph["ops"]:
        holder_of[op["output"]] = add({
            "kind": "sub_op", "device": 0, "tensor": op["output"], "op": op["id"],
            "phase": op["id"] + ":out", "region": [[0, e] for e in shapes[op["output"]]],
            "sources": [holder_of[i] for i in op["inputs"]]})
    for t in sorted(shapes):
        holders[t] = [holder_of[t]]
    return json.dumps({"k": 0, "devices": 1, "graph": graph, "assignment": {t: "phi" for t in shapes},
                       "hierarchy": {"levels": []}, "nodes": nodes, "holders": holders,
                       "fetch_bytes_total": 0})


def execute_numeric_host(plan_json: str, seed: int, ctx: Optional[Context] = None,
                         precision: int = PREC_TF32, flags: int = FLAG_FUSE) -> NumericCheck:
    """The same check with the comparison on the host (every holder read back): cross-checks the
    device reduction in the tests."""
    ctx = ctx or Context(0)
    plan = json.loads(plan_json)
    tiled = PlanExecutor(ctx, plan_json, precision, flags)
    serial = PlanExecutor(ctx, serial_plan(plan["graph"]), precision, flags)
    for ex in (tiled, serial):
        ex.init_inputs(seed)
        ex.execute()
        ex.synchronize()
    c = NumericCheck(seed=seed)
    nodes = {n["id"]: n for n in plan["nodes"]}
    for tid, hs in plan["holders"].items():
        full = serial.read_node(serial.holders()[tid][0])
        for d, hid in enumerate(hs):
            if d not in tiled.my_devices():
                continue
            reg = nodes[hid]["region"]
            want = full[tuple(slice(lo, hi) for lo, hi in reg)]
            diff = np.abs(tiled.read_node(hid) - want)
            if diff.size:
                c.max_abs = max(c.max_abs, float(diff.max()))
                c.max_rel = max(c.max_rel, float((diff / np.maximum(np.abs(want), 1.0)).max()))
            c.values += diff.size
    tiled.close()
    serial.close()
    return c


def execute_numeric(plan_json: str, seed: int, ctx: Optional[Context] = None,
                    precision: int = PREC_TF32, flags: int = FLAG_FUSE) -> NumericCheck:
    """B200 counterpart of execute_numeric (simulator.cpp:55-149): the tiled plan and the
    single-device run both execute on this GPU; every holder block of every tensor on every
    device is compared.  Multi-rank (ctx.world > 1): each rank checks the holders of its own
    logical devices; the single-device truth runs on a world-1 context of the same GPU."""
    ctx = ctx or Context(0)
    plan = json.loads(plan_json)
    tiled = PlanExecutor(ctx, plan_json, precision, flags)
    if ctx.world > 1 and (flags & FLAG_PEER):
        tiled.connect_peers_from_torch()
    solo = ctx if ctx.world == 1 else Context(ctx.ordinal, 0, 1)
    serial = PlanExecutor(solo, serial_plan(plan["graph"]), precision, flags & ~(FLAG_PEER | FLAG_FORCE_XCHG))
    tiled.init_inputs(seed)
    serial.init_inputs(seed)
    tiled.execute()
    serial.execute()
    tiled.synchronize()
    serial.synchronize()
    # the comparison runs on the device (tpx_numeric_check): one reduction over
    # every holder block of this rank; only max |d|, max rel and the count come back
    ma, mr, nv = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    check(lib().tpx_numeric_check(tiled._h, serial._h, ctypes.byref(ma), ctypes.byref(mr), ctypes.byref(nv)))
    c = NumericCheck(max_abs=ma.value, max_rel=mr.value, values=nv.value, seed=seed)
    tiled.close()
    serial.close()
    return c
