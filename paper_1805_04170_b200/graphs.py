"""Graph-JSON generators for the AlexNet- and VGG-style BASELINE configs.

The reference IR (proj/include/tileplan/graph.hpp) has stride-1 valid convolutions, matmuls and
elementwise ops only -- no pooling, padding or flatten -- and its `gen_cnn`
(proj/src/graph.cpp:231-314) takes one filter size for every layer and emits no weight update.
These generators write the same graph JSON the reference parses (`parse_graph`,
graph.cpp:405), op for op in gen_cnn's order and attribute layout, with per-layer filters and
the SGD update that gen_mlp emits (step = scale(lr), upd = sub, graph.cpp:217-227), so the
unchanged planner (kcuts / preset_assignment -> build_execution_graph) plans them.

A network is two components, planned and executed as two plans per train step (the IR cannot
express the flatten between them, SURVEY finding 7):
  * conv component: conv chain on [N, C, H, W] images (this module);
  * FC component: the reference's own gen_mlp over [N, C*H*W] (oracle.ref.gen_mlp /
    tools/make_plans.py).
"""
from __future__ import annotations

import json
from typing import List, Sequence, Tuple

# contraction-role attributes exactly as gen_cnn writes them (graph.cpp:231-314)
_CONV_ATTRS = {
    "forward": {"col_dims": [0, 1], "inner_dims": [1, 1], "row_dims": [0, 0]},
    "grad_weight": {"col_dims": [1, 0], "inner_dims": [0, 0], "row_dims": [1, 1]},
    "grad_input": {"col_dims": [1, 1], "inner_dims": [1, 0], "row_dims": [0, 0]},
}


def conv_net(batch: int, image_hw: Tuple[int, int], channels: Sequence[int],
             filters: Sequence[Tuple[int, int]], backward: bool = True, update: bool = True,
             lr: float = 0.01, dtype_bytes: int = 4) -> str:
    """One SGD train step of a stride-1 valid conv chain with tanh activations.

    channels = [C0, C1, ..., CL] (C0 = image channels), filters = [(U1, V1), ..., (UL, VL)].
    Tensor and op names follow gen_cnn (a<l>, k<l>, z<l>, g<l>, gk<l>, h<l>, fwd<l>, act<l>,
    seed, bwd_k<l>, bwd_a<l>, dact<l>) plus gen_mlp's update names (kd<l>, k<l>_next,
    step<l>, upd<l>)."""
    L = len(channels) - 1
    if L < 1 or len(filters) != L:
        raise ValueError("need one filter size per conv layer")
    tensors, ops = {}, []

    def tensor(tid, shape, role):
        tensors[tid] = {"dtype_bytes": dtype_bytes, "id": tid, "role": role, "shape": list(shape)}

    def conv(oid, mode, a, b, out):
        ops.append({"attrs": dict(_CONV_ATTRS[mode], mode=mode), "id": oid, "inputs": [a, b],
                    "kind": "conv", "output": out})

    def ew(oid, fn, ins, out, scale=None):
        attrs = {"function": fn}
        if scale is not None:
            attrs["scale"] = scale
        ops.append({"attrs": attrs, "id": oid, "inputs": list(ins), "kind": "elementwise", "output": out})

    H, W = image_hw
    hw = [(H, W)]
    for (u, v) in filters:
        H, W = H - u + 1, W - v + 1
        if H < 1 or W < 1:
            raise ValueError("image too small for the filter chain (valid convolutions)")
        hw.append((H, W))
    tensor("a0", (batch, channels[0]) + hw[0], "input")
    for l in range(1, L + 1):
        tensor(f"k{l}", (channels[l], channels[l - 1]) + tuple(filters[l - 1]), "weight")
        tensor(f"z{l}", (batch, channels[l]) + hw[l], "activation")
        tensor(f"a{l}", (batch, channels[l]) + hw[l], "activation")
        conv(f"fwd{l}", "forward", f"a{l - 1}", f"k{l}", f"z{l}")
        ew(f"act{l}", "pointwise_fn", [f"z{l}"], f"a{l}")
    if backward:
        tensor(f"g{L}", (batch, channels[L]) + hw[L], "gradient")
        ew("seed", "pointwise_fn_grad", [f"a{L}"], f"g{L}")
        for l in range(L, 0, -1):
            tensor(f"gk{l}", (channels[l], channels[l - 1]) + tuple(filters[l - 1]), "gradient")
            tensor(f"h{l - 1}", (batch, channels[l - 1]) + hw[l - 1], "gradient")
            conv(f"bwd_k{l}", "grad_weight", f"a{l - 1}", f"g{l}", f"gk{l}")
            conv(f"bwd_a{l}", "grad_input", f"g{l}", f"k{l}", f"h{l - 1}")
            if l > 1:
                tensor(f"g{l - 1}", (batch, channels[l - 1]) + hw[l - 1], "gradient")
                ew(f"dact{l - 1}", "pointwise_fn_grad", [f"h{l - 1}"], f"g{l - 1}")
        if update:
            for l in range(1, L + 1):
                shape = (channels[l], channels[l - 1]) + tuple(filters[l - 1])
                tensor(f"kd{l}", shape, "temp")
                tensor(f"k{l}_next", shape, "weight")
                ew(f"step{l}", "scale", [f"gk{l}"], f"kd{l}", scale=lr)
                ew(f"upd{l}", "sub", [f"k{l}", f"kd{l}"], f"k{l}_next")
    g = {"ops": ops, "tensors": [tensors[k] for k in sorted(tensors)]}
    return json.dumps(g, sort_keys=True)


# BASELINE configs[2] / configs[3] conv components (stated shapes; SURVEY §8(d) "Synthetic
# inputs"): stride-1 valid convolutions only, so the images are chosen to end at the FC
# component's input width.
ALEXNET_CONV = {"image_hw": (48, 48), "channels": [3, 96, 256, 384, 384, 256],
                "filters": [(11, 11), (5, 5), (3, 3), (3, 3), (3, 3)]}        # -> 256 x 28 x 28
VGG_CONV = {"image_hw": (33, 33),
            "channels": [3, 64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512],
            "filters": [(3, 3)] * 13}                                           # -> 512 x 7 x 7 = 25088
ALEXNET_FC = [9216, 4096, 4096, 1000]
VGG_FC = [25088, 4096, 4096, 1000]


def alexnet_conv(batch: int, **kw) -> str:
    return conv_net(batch, ALEXNET_CONV["image_hw"], ALEXNET_CONV["channels"], ALEXNET_CONV["filters"], **kw)


def vgg_conv(batch: int, **kw) -> str:
    return conv_net(batch, VGG_CONV["image_hw"], VGG_CONV["channels"], VGG_CONV["filters"], **kw)


def conv_flops(graph_json: str) -> float:
    """Algorithmic FLOPs of the graph's convolutions: 2 * |out| * contraction."""
    g = json.loads(graph_json)
    sh = {t["id"]: t["shape"] for t in g["tensors"]}
    f = 0.0
    for op in g["ops"]:
        if op["kind"] != "conv":
            continue
        a, b, o = sh[op["inputs"][0]], sh[op["inputs"][1]], sh[op["output"]]
        mode = op["attrs"]["mode"]
        n_out = o[0] * o[1] * o[2] * o[3]
        if mode == "forward":
            f += 2.0 * n_out * b[1] * b[2] * b[3]
        elif mode == "grad_weight":
            f += 2.0 * n_out * a[0] * b[2] * b[3]
        else:  # grad_input: taps inside the gradient only (the reference's bounds-checked sum)
            f += 2.0 * a[0] * a[1] * a[2] * a[3] * b[1] * b[2] * b[3]
    return f
