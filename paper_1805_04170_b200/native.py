"""ctypes binding of the native library (include/tpx.h).

The library is built in-tree by `paper_1805_04170_b200/build.py` (or `__graft_entry__.build()`).
There is no fallback: if `_lib/libtpx.so` is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_lib", "libtpx.so")

_lib = None

P = ctypes.POINTER
c_i64, c_int, c_u64, c_dbl, c_vp, c_char_p = (ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                              ctypes.c_double, ctypes.c_void_p, ctypes.c_char_p)


class TpxError(RuntimeError):
    """An error reported by the native library (mirrors tileplan::Error)."""


class Stats(ctypes.Structure):
    _fields_ = [
        ("fetch_bytes_total", c_i64), ("rank_fetch_bytes_in", c_i64),
        ("rank_xrank_bytes_in", c_i64), ("rank_xrank_bytes_out", c_i64), ("n_nodes", c_i64),
        ("n_steps", c_i64), ("n_kernel_launches", c_i64), ("n_gemm_launches", c_i64),
        ("n_copy_launches", c_i64), ("n_nccl_groups", c_i64), ("n_fused_ew", c_i64),
        ("device_bytes", c_i64), ("gemm_flops", c_dbl), ("gemm_min_bytes", c_dbl),
        ("storage_bytes", c_i64),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


# Declared signatures: name -> (argtypes).  restype is int (status) unless noted.
_SIGS = {
    "tpx_version": [],
    "tpx_create": [c_int, c_int, c_int, P(c_vp)],
    "tpx_init_comm": [c_vp, c_vp, ctypes.c_size_t],
    "tpx_comm_unique_id": [c_vp, ctypes.c_size_t],
    "tpx_destroy": [c_vp],
    "tpx_load_plan": [c_vp, c_char_p, ctypes.c_size_t, c_int, c_int, P(c_vp)],
    "tpx_plan_free": [c_vp],
    "tpx_plan_ipc_handle": [c_vp, c_vp, ctypes.c_size_t],
    "tpx_numeric_check": [c_vp, c_vp, P(c_dbl), P(c_dbl), P(c_i64)],
    "tpx_plan_connect_peers": [c_vp, c_vp, ctypes.c_size_t],
    "tpx_plan_stats": [c_vp, P(Stats)],
    "tpx_plan_describe": [c_vp, P(c_vp)],
    "tpx_init_inputs": [c_vp, c_u64],
    "tpx_node_elements": [c_vp, c_char_p, P(c_i64)],
    "tpx_write_node": [c_vp, c_char_p, P(c_dbl), c_i64],
    "tpx_read_node": [c_vp, c_char_p, P(c_dbl), c_i64],
    "tpx_write_node_f32": [c_vp, c_char_p, c_vp, c_i64],
    "tpx_read_node_f32": [c_vp, c_char_p, c_vp, c_i64],
    "tpx_node_view": [c_vp, c_char_p, P(c_u64), P(c_int), P(c_i64), P(c_i64)],
    "tpx_set_stream": [c_vp, c_u64],
    "tpx_execute": [c_vp],
    "tpx_execute_op": [c_vp, c_char_p],
    "tpx_carry_weights": [c_vp],
    "tpx_synchronize": [c_vp],
    "tpx_last_timing": [c_vp, P(c_dbl), P(c_dbl), P(c_dbl)],
    "tpx_enable_timing": [c_vp, c_int],
    "tpx_last_step_times": [c_vp, P(c_dbl), c_i64, P(c_i64)],
    "tpx_execute_steps": [c_vp, c_i64, c_i64],
    "tpx_copy_node_device": [c_vp, c_char_p, c_vp, c_i64, c_int],
    "tpx_gemm": [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_vp, c_i64,
                 c_int, P(c_int), P(ctypes.c_float), P(c_vp), P(c_i64), P(c_vp), P(c_i64), c_int,
                 c_u64],
    "tpx_gemm_timed": [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_vp,
                       c_i64, c_int, P(c_int), P(ctypes.c_float), P(c_vp), P(c_i64), P(c_vp),
                       P(c_i64), c_int, c_u64, c_int, c_int, P(c_dbl)],
    "tpx_gemm_schedule": [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, P(c_int), P(c_int),
                          P(c_int), P(c_int), P(c_int), P(ctypes.c_int32), c_int,
                          P(ctypes.c_int32), c_int],
    "tpx_debug_gemm_mn_desc": [ctypes.c_uint, ctypes.c_uint],
    "tpx_debug_gemm_trace": [P(c_u64), c_int],
    "tpx_gemm_last_launch": [P(c_i64), c_int],
}


def exported_symbols():
    """Every entry point include/tpx.h declares (used by the symbol-export test)."""
    return sorted(list(_SIGS) + ["tpx_last_error", "tpx_free_string"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TpxError(f"native library missing: {LIB_PATH} — run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.tpx_last_error.restype = c_char_p
        if hasattr(L, "tpx_free_string"):
            L.tpx_free_string.argtypes = [c_vp]
            L.tpx_free_string.restype = None
        for name, args in _SIGS.items():
            if not hasattr(L, name):
                continue  # reported by the export test; calling it raises AttributeError
            f = getattr(L, name)
            f.argtypes = args
            f.restype = c_int
        _lib = L
    return _lib


def check(status: int):
    if status != 0:
        raise TpxError(lib().tpx_last_error().decode())


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def gemm(A, B, ta: bool, tb: bool, C, epi=None, stream=None, precision: int = 0,
         warmup: int = 0, iters: int = 0):
    """C = op(A) @ op(B) on the tcgen05 path; A, B, C are 2-D fp32 CUDA tensors with unit
    inner stride.  `epi` = [(op, scale, other_or_None, out), ...] (gemm.h EpiOp codes).
    With iters > 0 the prepared launch runs `warmup` + `iters` times and the mean device time
    (ms, CUDA events on the stream) is returned."""
    import torch  # plumbing only: device pointers and the current stream

    want = torch.bfloat16 if precision == 2 else torch.float32
    for t in (A, B, C):
        if t.dtype != want or t.dim() != 2 or t.stride(1) != 1:
            raise TpxError(f"gemm operands must be 2-D {want} with unit inner stride")
    epi = epi or []
    n = len(epi)
    ops = (c_int * max(n, 1))(*[e[0] for e in epi])
    scales = (ctypes.c_float * max(n, 1))(*[e[1] for e in epi])
    others = (c_vp * max(n, 1))(*[(e[2].data_ptr() if e[2] is not None else 0) for e in epi])
    others_rs = (c_i64 * max(n, 1))(*[(e[2].stride(0) if e[2] is not None else 0) for e in epi])
    outs = (c_vp * max(n, 1))(*[e[3].data_ptr() for e in epi])
    outs_rs = (c_i64 * max(n, 1))(*[e[3].stride(0) for e in epi])
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    ms = c_dbl(0.0)
    check(lib().tpx_gemm_timed(_ptr(A), A.shape[0], A.shape[1], A.stride(0), _ptr(B), B.shape[0],
                               B.shape[1], B.stride(0), int(ta), int(tb), _ptr(C), C.stride(0), n,
                               ops, scales, others, others_rs, outs, outs_rs, int(precision), s,
                               int(warmup), int(iters), ctypes.byref(ms)))
    return ms.value if iters > 0 else None


LAUNCH_FIELDS = ("bn", "pair", "swap", "p_mn", "q_mn", "oloader", "other_smem", "stream_k", "group",
                 "tstore", "nbox", "odepth", "stages", "units", "split", "bf16")


def last_launch():
    """The kernel variant the last gemm() call on this thread launched (tpx_gemm_last_launch)."""
    buf = (c_i64 * 16)()
    check(lib().tpx_gemm_last_launch(buf, 16))
    return dict(zip(LAUNCH_FIELDS, list(buf)))


def gemm_schedule(nprob: int, P_: int, Q: int, K: int, bn: int, num_sms: int = 148,
                  force_groups: int = 0, max_kb: int = 0):
    """Host-only view of the persistent GEMM's tile schedule (gemm.cu gemm_schedule):
    returns dict(grid, group, stream_k, nslots, segs=[(prob,tp,tq,kb0,kb1,kind,slot,n_parts)],
    seg_off=[...])."""
    grid, nsegs, nslots, group, sk = (c_int(), c_int(), c_int(), c_int(), c_int())
    check(lib().tpx_gemm_schedule(nprob, P_, Q, K, bn, num_sms, force_groups, max_kb, ctypes.byref(grid),
                                  ctypes.byref(nsegs), ctypes.byref(nslots), ctypes.byref(group),
                                  ctypes.byref(sk), None, 0, None, 0))
    segs = (ctypes.c_int32 * (8 * max(nsegs.value, 1)))()
    off = (ctypes.c_int32 * (grid.value + 1))()
    check(lib().tpx_gemm_schedule(nprob, P_, Q, K, bn, num_sms, force_groups, max_kb, ctypes.byref(grid),
                                  ctypes.byref(nsegs), ctypes.byref(nslots), ctypes.byref(group),
                                  ctypes.byref(sk), segs, nsegs.value, off, grid.value))
    return {"grid": grid.value, "group": group.value, "stream_k": bool(sk.value),
            "nslots": nslots.value,
            "segs": [tuple(segs[8 * i: 8 * i + 8]) for i in range(nsegs.value)],
            "seg_off": list(off)}
