"""Zero-copy torch views of executor node values (tpx_node_view) for the full-size GPU tests:
oracle values are copied straight into holder blocks on the device and node values are read
without host round trips.  Test plumbing only."""
import torch


class _CAI:
    def __init__(self, ptr, shape, strides_bytes, typestr):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "strides": tuple(strides_bytes), "typestr": typestr,
                                         "version": 3}


def node_tensor(ex, node_id):
    """The node's value on the device, in the plan's storage type (fp32 or bf16), as a strided
    torch view into the executor's arena."""
    ptr, shape, st = ex.node_view(node_id)
    es = ex.storage_bytes()
    if not shape:
        shape, st = [1], [1]
    strides = [s * es if n > 1 else es for s, n in zip(st, shape)]
    t = torch.as_tensor(_CAI(ptr, shape, strides, "<f4" if es == 4 else "<i2"), device="cuda")
    return t if es == 4 else t.view(torch.bfloat16)


def put(ex, node_id, value):
    """Write an fp64 value into a node's block (rounded fp64 -> fp32 [-> bf16], like
    tpx_write_node)."""
    t = node_tensor(ex, node_id)
    v = value.to(device="cuda", dtype=torch.float32)
    t.copy_(v.to(t.dtype))
    # the executor runs on its own stream: the value must land before its next launch reads it
    torch.cuda.synchronize()


def get(ex, node_id):
    return node_tensor(ex, node_id).double()


def normwise(got, want):
    if got.numel() == 0:
        return 0.0
    return ((got.double() - want.double()).abs().max() / want.double().abs().max().clamp_min(1e-30)).item()
