"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's CPU tiled executor.

This is the checker, never the thing measured or shipped: only tests/, tools/,
`__graft_entry__.smoke()` and bench.py's cpu_baseline leg import it.  The product path
(paper_1805_04170_b200) must not import or call anything under oracle/.

Restated (fp64, row-major, same semantics; vectorised instead of per-element loops):
  seeded_tensor     proj/src/dense.cpp:30-57   splitmix64 keyed by seed ^ FNV-1a(tensor id)
  bindings          proj/src/dense.cpp:59-67   tanh and 1 - tanh^2
  run_matmul        proj/src/dense.cpp:71-90
  run_conv          proj/src/dense.cpp:92-157  forward / grad_weight / grad_input, stride 1, valid
  run_op_dense      proj/src/dense.cpp:161-209 elementwise add/sub/scale/fn/fn_grad
  extract/paste     proj/src/dense.cpp:213-259 N-d box copy (+ accumulate)
  serial_execute    proj/src/oracle.cpp:176-202
  execute_numeric   proj/src/simulator.cpp:55-149 node interpreter + max_abs / max_rel check
  simulate_traffic  proj/src/simulator.cpp:11-49 (byte accounting only)

Pinned by tests/test_oracle.py against (a) golden fixtures in tests/golden/ produced by the
compiled reference itself (tools/make_golden.py via oracle/_ref) and (b) the reference's
own known-answer cases (proj/tests/test_plan.cpp:178-223, acceptance.cpp:277-293).
Matmul sums use BLAS order rather than the reference's sequential p-loop; the difference is
at the 1e-15 relative level, far inside the reference's own 1e-12 gate (main.cpp:361).
"""
from __future__ import annotations

import json
from typing import Dict, List

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def fnv1a(s: str) -> int:
    """dense.cpp:38-45."""
    h = 0xCBF29CE484222325
    for c in s.encode():
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def seeded_values(n: int, seed: int, tensor_id: str, start: int = 0) -> np.ndarray:
    """Elements [start, start+n) of seeded_tensor's row-major stream (dense.cpp:49-57).

    splitmix64 advances its state by the golden gamma before mixing, so element i uses
    state0 + (i+1)*gamma; the top 53 bits map to [-1, 1) exactly as the reference does."""
    s0 = np.uint64((seed ^ fnv1a(tensor_id)) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = s0 + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    bits = (z >> np.uint64(11)).astype(np.float64)
    return bits * (2.0 / 9007199254740992.0) - 1.0


def seeded_tensor(shape, seed: int, tensor_id: str) -> np.ndarray:
    n = int(np.prod(shape)) if len(shape) else 1
    return seeded_values(n, seed, tensor_id).reshape(shape)


# ---------------------------------------------------------------- kernels (dense.cpp)

def run_matmul(attrs: dict, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """dense.cpp:71-90: out = op(A) @ op(B) with transpose flags."""
    A = a.T if attrs.get("transpose_a", False) else a
    B = b.T if attrs.get("transpose_b", False) else b
    if A.shape[1] != B.shape[0]:
        raise ValueError("matmul inner extents differ")
    return A @ B


def run_conv(attrs: dict, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """dense.cpp:92-157 (stride 1, valid; grad_input is the full correlation)."""
    mode = attrs["mode"]
    if mode == "forward":
        n, ci, h, w = a.shape
        co, ci2, fh, fw = b.shape
        ho, wo = h - fh + 1, w - fw + 1
        out = np.zeros((n, co, ho, wo))
        for u in range(fh):
            for v in range(fw):
                out += np.einsum("nchw,oc->nohw", a[:, :, u:u + ho, v:v + wo], b[:, :, u, v])
        return out
    if mode == "grad_weight":
        n, ci, h, w = a.shape
        _, co, ho, wo = b.shape
        fh, fw = h - ho + 1, w - wo + 1
        out = np.zeros((co, ci, fh, fw))
        for u in range(fh):
            for v in range(fw):
                out[:, :, u, v] = np.einsum("nchw,nohw->oc", a[:, :, u:u + ho, v:v + wo], b)
        return out
    # grad_input: A = G (n, co, ho, wo), B = K (co, ci, fh, fw)
    n, co, ho, wo = a.shape
    _, ci, fh, fw = b.shape
    out = np.zeros((n, ci, ho + fh - 1, wo + fw - 1))
    for u in range(fh):
        for v in range(fw):
            out[:, :, u:u + ho, v:v + wo] += np.einsum("nohw,oc->nchw", a, b[:, :, u, v])
    return out


def fn(x):
    return np.tanh(x)


def fn_grad(x):
    t = np.tanh(x)
    return 1.0 - t * t


def run_op_dense(op: dict, inputs: List[np.ndarray]) -> np.ndarray:
    """dense.cpp:161-209."""
    kind = op["kind"]
    attrs = op.get("attrs", {})
    if kind == "matmul":
        return run_matmul(attrs, inputs[0], inputs[1])
    if kind == "conv":
        return run_conv(attrs, inputs[0], inputs[1])
    if kind == "elementwise":
        f = attrs["function"]
        for x in inputs:
            if x.shape != inputs[0].shape:
                raise ValueError(f"op '{op['id']}': elementwise operands must share a shape")
        if f == "add":
            return inputs[0] + inputs[1]
        if f == "sub":
            return inputs[0] - inputs[1]
        if f == "scale":
            return attrs.get("scale", 0.0) * inputs[0]
        if f == "pointwise_fn":
            return fn(inputs[0])
        if f == "pointwise_fn_grad":
            return fn_grad(inputs[0])
    raise ValueError(f"op '{op['id']}': unbound function tag (generic ops have no numeric binding)")


# ---------------------------------------------------------------- regions (dense.cpp:213-259)

def region_slices(region, within) -> tuple:
    return tuple(slice(lo - w0, hi - w0) for (lo, hi), (w0, _) in zip(region, within))


def region_volume(region) -> int:
    v = 1
    for lo, hi in region:
        if hi <= lo:
            return 0
        v *= hi - lo
    return v


def region_shape(region):
    return [hi - lo for lo, hi in region]


def extract_region(src: np.ndarray, src_region, sub) -> np.ndarray:
    for (lo, hi), (s0, s1) in zip(sub, src_region):
        if lo < s0 or hi > s1:
            raise ValueError("slice region escapes source region")
    return src[region_slices(sub, src_region)].copy()


def paste_region(dst: np.ndarray, dst_region, piece: np.ndarray, piece_region, accumulate: bool):
    for (lo, hi), (d0, d1) in zip(piece_region, dst_region):
        if lo < d0 or hi > d1:
            raise ValueError("piece region escapes destination region")
    sl = region_slices(piece_region, dst_region)
    if accumulate:
        dst[sl] += piece
    else:
        dst[sl] = piece


# ---------------------------------------------------------------- graph execution

def graph_inputs(graph: dict) -> List[str]:
    produced = {op["output"] for op in graph["ops"]}
    return [t["id"] for t in graph["tensors"] if t["id"] not in produced]


def serial_execute(graph: dict, seed: int, preset: Dict[str, np.ndarray] | None = None):
    """oracle.cpp:176-202: every tensor's full fp64 value."""
    shapes = {t["id"]: t["shape"] for t in graph["tensors"]}
    vals: Dict[str, np.ndarray] = {}
    for tid in graph_inputs(graph):
        vals[tid] = preset[tid] if preset and tid in preset else seeded_tensor(shapes[tid], seed, tid)
    for op in graph["ops"]:
        out = run_op_dense(op, [vals[i] for i in op["inputs"]])
        if list(out.shape) != list(shapes[op["output"]]):
            raise ValueError(f"op '{op['id']}' produced an unexpected shape")
        vals[op["output"]] = out
    return vals


def execute_nodes(plan: dict, serial: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
    """simulator.cpp:77-127: literal node-by-node interpretation, every node's block."""
    graph = plan["graph"]
    shapes = {t["id"]: t["shape"] for t in graph["tensors"]}
    ops = {op["id"]: op for op in graph["ops"]}
    vals: Dict[str, np.ndarray] = {}
    regions = {}
    for n in plan["nodes"]:
        kind, reg = n["kind"], n["region"]
        if kind == "buffer":
            full = [[0, e] for e in shapes[n["tensor"]]]
            v = extract_region(serial[n["tensor"]], full, reg)
        elif kind in ("slice", "fetch"):
            s = n["sources"][0]
            v = extract_region(vals[s], regions[s], reg)
        elif kind == "concat":
            v = np.zeros(region_shape(reg))
            pasted = 0
            for s in n["sources"]:
                paste_region(v, reg, vals[s], regions[s], False)
                pasted += region_volume(regions[s])
            if pasted != region_volume(reg):
                raise ValueError(f"concat node {n['id']} pieces do not tile its region")
        elif kind == "reduce_partial":
            v = np.zeros(region_shape(reg))
            for s in n["sources"]:
                if regions[s] != reg:
                    raise ValueError(f"reduce node {n['id']} sums mismatched regions")
                paste_region(v, reg, vals[s], regions[s], True)
        elif kind == "sub_op":
            v = run_op_dense(ops[n["op"]], [vals[s] for s in n["sources"]])
            if list(v.shape) != region_shape(reg):
                raise ValueError(f"sub-op node {n['id']} produced a mismatched block")
        else:
            raise ValueError(f"unknown node kind '{kind}'")
        vals[n["id"]] = v
        regions[n["id"]] = reg
    return vals


def numeric_check(plan: dict, serial, node_values) -> dict:
    """simulator.cpp:129-147: max |d| and max |d| / max(|ref|, 1) over every holder."""
    shapes = {t["id"]: t["shape"] for t in plan["graph"]["tensors"]}
    nodes = {n["id"]: n for n in plan["nodes"]}
    max_abs = max_rel = 0.0
    count = 0
    for tid, holders in plan["holders"].items():
        full = [[0, e] for e in shapes[tid]]
        for hid in holders:
            if not hid:
                raise ValueError(f"tensor {tid} has no holder on some device")
            want = extract_region(serial[tid], full, nodes[hid]["region"])
            d = np.abs(node_values[hid] - want)
            if d.size:
                max_abs = max(max_abs, float(d.max()))
                max_rel = max(max_rel, float((d / np.maximum(np.abs(want), 1.0)).max()))
            count += d.size
    return {"max_abs": max_abs, "max_rel": max_rel, "values": count}


def execute_numeric(plan, seed: int) -> dict:
    """simulator.cpp:55-149."""
    if isinstance(plan, str):
        plan = json.loads(plan)
    serial = serial_execute(plan["graph"], seed)
    vals = execute_nodes(plan, serial)
    c = numeric_check(plan, serial, vals)
    c["seed"] = seed
    return c


def fetch_bytes_by_phase(plan: dict) -> Dict[str, int]:
    """Per-phase fetch bytes (simulator.cpp:26-38 without the level attribution)."""
    out: Dict[str, int] = {}
    for n in plan["nodes"]:
        if n["kind"] == "fetch":
            out[n["phase"]] = out.get(n["phase"], 0) + int(n["bytes"])
    return out


def per_op_bytes(plan: dict) -> Dict[str, int]:
    """Fetch bytes grouped by op (phases '<op>:in<j>' and '<op>:out'); equals
    graph_cost(g, a).per_op[op].bytes (cost.cpp:244-253)."""
    out: Dict[str, int] = {op["id"]: 0 for op in plan["graph"]["ops"]}
    for n in plan["nodes"]:
        if n["kind"] == "fetch":
            op = n["phase"].rsplit(":", 1)[0]
            out[op] += int(n["bytes"])
    return out


def algorithmic_flops(graph: dict) -> int:
    """Sum of 2*M*N*K over matmuls and 2*|out|*contraction over convs."""
    shapes = {t["id"]: t["shape"] for t in graph["tensors"]}
    f = 0
    for op in graph["ops"]:
        if op["kind"] == "matmul":
            a = shapes[op["inputs"][0]]
            kk = a[0] if op["attrs"].get("transpose_a") else a[1]
            o = shapes[op["output"]]
            f += 2 * o[0] * o[1] * kk
        elif op["kind"] == "conv":
            a, b, o = (shapes[op["inputs"][0]], shapes[op["inputs"][1]], shapes[op["output"]])
            m = op["attrs"]["mode"]
            if m == "forward":       # every output element contracts ci*fh*fw taps
                f += 2 * int(np.prod(o)) * b[1] * b[2] * b[3]
            elif m == "grad_weight":  # every filter tap contracts n*ho*wo
                f += 2 * int(np.prod(o)) * a[0] * b[2] * b[3]
            else:                     # full correlation: each G element meets ci*fh*fw taps
                f += 2 * int(np.prod(a)) * b[1] * b[2] * b[3]
    return f
