"""TEST INFRASTRUCTURE ONLY — torch fp64 restatement of the reference's CPU tiled executor,
for the full-size parity tests (SURVEY §7 H5 / §8(c) parity plan item 4).

The reference's own executor (and oracle/tileplan_oracle.py, its numpy restatement) cannot
run the BASELINE configs at full size: cfg2 is ~1 TFLOP per step in fp64, hours on one core.
This module restates the same functions in torch fp64 so that the checker can run on the
GPU box's device (fp64 on the B200) or on CPU at small sizes.  It is the checker, never the
thing measured or shipped: only tests/ import it.

Restated (same semantics as tileplan_oracle, which cites the reference lines):
  seeded_tensor     proj/src/dense.cpp:30-57    splitmix64 keyed by seed ^ FNV-1a(id), in int64
                                                 arithmetic (wrapping), bit-exact
  run_matmul        proj/src/dense.cpp:71-90
  run_conv          proj/src/dense.cpp:92-157   forward = conv2d, grad_weight = conv2d over the
                                                 batch, grad_input = conv_transpose2d (the full
                                                 correlation), stride 1, valid
  run_op_dense      proj/src/dense.cpp:161-209
  serial_execute    proj/src/oracle.cpp:176-202
  execute_nodes     proj/src/simulator.cpp:77-127 (slices/fetches are views: node values are
                                                 immutable in the interpreter)

Pinned by tests/test_torch_oracle.py against the golden fixtures produced by the compiled
reference (bit-exact seeded inputs; values within 1e-10 like the numpy restatement).
"""
from __future__ import annotations

import json
from typing import Dict, List

import torch
import torch.nn.functional as F

from oracle.tileplan_oracle import fnv1a


def _s64(x: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    x &= 0xFFFFFFFFFFFFFFFF
    return x - (1 << 64) if x >= 1 << 63 else x


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_M1 = _s64(0xBF58476D1CE4E5B9)
_M2 = _s64(0x94D049BB133111EB)


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def seeded_tensor(shape, seed: int, tensor_id: str, device="cpu", chunk: int = 1 << 25) -> torch.Tensor:
    """dense.cpp:49-57: element i (row-major) = splitmix64(state0 + (i+1)*gamma) >> 11 mapped to
    [-1, 1) exactly (53-bit integers are exact in fp64)."""
    n = 1
    for e in shape:
        n *= int(e)
    s0 = _s64(seed ^ fnv1a(tensor_id))
    out = torch.empty(n, dtype=torch.float64, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        i = torch.arange(a + 1, b + 1, dtype=torch.int64, device=device)
        z = i * _GOLDEN + s0
        z = (z ^ _srl(z, 30)) * _M1
        z = (z ^ _srl(z, 27)) * _M2
        z = z ^ _srl(z, 31)
        out[a:b] = _srl(z, 11).to(torch.float64) * (2.0 / 9007199254740992.0) - 1.0
    return out.reshape([int(e) for e in shape])


def run_matmul(attrs: dict, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    A = a.t() if attrs.get("transpose_a", False) else a
    B = b.t() if attrs.get("transpose_b", False) else b
    if A.shape[1] != B.shape[0]:
        raise ValueError("matmul inner extents differ")
    return A @ B


def run_conv(attrs: dict, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    mode = attrs["mode"]
    if mode == "forward":        # out[n,o,y,x] = sum_{c,u,v} A[n,c,y+u,x+v] K[o,c,u,v]
        return F.conv2d(a, b)
    if mode == "grad_weight":    # out[o,c,u,v] = sum_{n,y,x} A[n,c,y+u,x+v] G[n,o,y,x]
        return F.conv2d(a.transpose(0, 1), b.transpose(0, 1)).transpose(0, 1).contiguous()
    # grad_input: out[n,c,y,x] = sum_{o,u,v} G[n,o,y-u,x-v] K[o,c,u,v]
    return F.conv_transpose2d(a, b)


def fn(x):
    return torch.tanh(x)


def fn_grad(x):
    t = torch.tanh(x)
    return 1.0 - t * t


def run_op_dense(op: dict, inputs: List[torch.Tensor]) -> torch.Tensor:
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


def graph_inputs(graph: dict) -> List[str]:
    produced = {op["output"] for op in graph["ops"]}
    return [t["id"] for t in graph["tensors"] if t["id"] not in produced]


def serial_execute(graph: dict, seed: int, device="cpu", dtype=torch.float64,
                   inputs: Dict[str, torch.Tensor] | None = None) -> Dict[str, torch.Tensor]:
    """oracle.cpp:176-202.  dtype=float32 gives the plain-fp32 execution of the same graph (the
    measured fp32 floor the chained gates are stated against)."""
    shapes = {t["id"]: t["shape"] for t in graph["tensors"]}
    vals: Dict[str, torch.Tensor] = {}
    for tid in graph_inputs(graph):
        v = inputs[tid] if inputs and tid in inputs else seeded_tensor(shapes[tid], seed, tid, device)
        vals[tid] = v.to(dtype)
    for op in graph["ops"]:
        out = run_op_dense(op, [vals[i] for i in op["inputs"]])
        if list(out.shape) != list(shapes[op["output"]]):
            raise ValueError(f"op '{op['id']}' produced an unexpected shape")
        vals[op["output"]] = out
    return vals


def _slices(region, within):
    return tuple(slice(lo - w0, hi - w0) for (lo, hi), (w0, _) in zip(region, within))


def execute_nodes(plan: dict, serial: Dict[str, torch.Tensor]) -> Dict[str, torch.Tensor]:
    """simulator.cpp:77-127: every node's block (views where the interpreter copies)."""
    graph = plan["graph"]
    shapes = {t["id"]: t["shape"] for t in graph["tensors"]}
    ops = {op["id"]: op for op in graph["ops"]}
    vals: Dict[str, torch.Tensor] = {}
    regions = {}
    for n in plan["nodes"]:
        kind, reg = n["kind"], n["region"]
        if kind == "buffer":
            v = serial[n["tensor"]][_slices(reg, [[0, e] for e in shapes[n["tensor"]]])]
        elif kind in ("slice", "fetch"):
            s = n["sources"][0]
            v = vals[s][_slices(reg, regions[s])]
        elif kind in ("concat", "reduce_partial"):
            ref = vals[n["sources"][0]]
            v = torch.zeros([hi - lo for lo, hi in reg], dtype=ref.dtype, device=ref.device)
            for s in n["sources"]:
                if kind == "reduce_partial":
                    if regions[s] != reg:
                        raise ValueError(f"reduce node {n['id']} sums mismatched regions")
                    v += vals[s]
                else:
                    v[_slices(regions[s], reg)] = vals[s]
        elif kind == "sub_op":
            v = run_op_dense(ops[n["op"]], [vals[s] for s in n["sources"]])
        else:
            raise ValueError(f"unknown node kind '{kind}'")
        vals[n["id"]] = v
        regions[n["id"]] = reg
    return vals


def load(plan_json: str) -> dict:
    return json.loads(plan_json)
