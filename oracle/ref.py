"""TEST INFRASTRUCTURE ONLY — ctypes access to the unmodified reference library.

`oracle/_ref/libtileplan_ref.so` is the reference planner + CPU tiled executor compiled from
/root/reference/proj/src by `oracle/Makefile`, plus `oracle/ref_driver.cpp` (extern "C"
entry points over the reference's public API).  Only tests/, tools/ (fixture generation),
`__graft_entry__.smoke()` and bench.py's CPU-baseline / `--impl reference` legs may use it.
The product path (paper_1805_04170_b200) never imports this module.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtileplan_ref.so")

_lib = None


def build(quiet: bool = True) -> bool:
    """Compile oracle/_ref from /root/reference if that tree exists (only in the build
    container).  Returns True when the library is present afterwards."""
    if os.path.isdir("/root/reference/proj/src"):
        # the library, and INTEGRATION.md's reference-side adapter linked against libtpx.so
        # (integration/*.cpp -> oracle/_ref/adapter_b200; needs the product library built first)
        out = subprocess.run(["make", "-C", HERE, "-j8", "all", "adapter"], capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError("oracle/_ref build failed:\n" + out.stdout + out.stderr)
    return os.path.exists(LIB_PATH)


ADAPTER = os.path.join(HERE, "_ref", "adapter_b200")


def available() -> bool:
    return os.path.exists(LIB_PATH)


class RefError(RuntimeError):
    """Mirror of tileplan::Error crossing the driver's C boundary."""


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"reference library not built: {LIB_PATH} (run make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        c_char_p, c_int, c_i64, c_u64, c_dbl = (ctypes.c_char_p, ctypes.c_int, ctypes.c_int64,
                                                ctypes.c_uint64, ctypes.c_double)
        P = ctypes.POINTER
        L.ref_last_error.restype = c_char_p
        L.ref_free.argtypes = [ctypes.c_void_p]
        for name, args in {
            "ref_gen_mlp": [c_i64, P(c_i64), c_int, c_int, c_int, c_dbl, c_int],
            "ref_gen_cnn": [c_i64, c_i64, c_i64, P(c_i64), c_int, c_i64, c_i64, c_int, c_int],
            "ref_assignment": [c_char_p, c_char_p, c_int],
            "ref_kcuts": [c_char_p, c_int],
            "ref_graph_cost": [c_char_p, c_char_p, c_int],
            "ref_plan": [c_char_p, c_char_p, c_int, c_char_p],
            "ref_plan_roundtrip": [c_char_p],
            "ref_simulate_traffic": [c_char_p, c_char_p],
        }.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_void_p
        L.ref_execute_numeric.argtypes = [c_char_p, c_u64, P(c_dbl), P(c_dbl), P(c_i64), P(c_dbl)]
        L.ref_execute_numeric_parallel.argtypes = [c_char_p, c_u64, c_int, P(c_dbl)]
        L.ref_serial_seconds.argtypes = [c_char_p, c_u64, P(c_dbl)]
        L.ref_session_new.argtypes = [c_char_p, c_u64]
        L.ref_session_new.restype = ctypes.c_void_p
        L.ref_session_free.argtypes = [ctypes.c_void_p]
        L.ref_session_times.argtypes = [ctypes.c_void_p, P(c_dbl), P(c_dbl)]
        L.ref_session_serial.argtypes = [ctypes.c_void_p, c_char_p, P(c_dbl), c_i64]
        L.ref_session_node.argtypes = [ctypes.c_void_p, c_char_p, P(c_dbl), c_i64]
        L.ref_pool_new.argtypes = [c_char_p, c_u64, c_int]
        L.ref_pool_new.restype = ctypes.c_void_p
        L.ref_pool_step.argtypes = [ctypes.c_void_p, P(c_dbl)]
        L.ref_pool_step.restype = c_int
        L.ref_pool_free.argtypes = [ctypes.c_void_p]
        for f in (L.ref_execute_numeric, L.ref_execute_numeric_parallel, L.ref_serial_seconds,
                  L.ref_session_times, L.ref_session_serial, L.ref_session_node):
            f.restype = c_int
        _lib = L
    return _lib


def _s(ptr) -> str:
    if not ptr:
        raise RefError(lib().ref_last_error().decode())
    try:
        return ctypes.string_at(ptr).decode()
    finally:
        lib().ref_free(ptr)


def _b(s) -> bytes:
    return s.encode() if isinstance(s, str) else s


def gen_mlp(batch, dims, backward=True, update=True, lr=0.01, dtype_bytes=4) -> str:
    arr = (ctypes.c_int64 * len(dims))(*dims)
    return _s(lib().ref_gen_mlp(batch, arr, len(dims), int(backward), int(update), lr, dtype_bytes))


def gen_cnn(batch, image_hw, channels, filter_hw, backward=True, dtype_bytes=4) -> str:
    arr = (ctypes.c_int64 * len(channels))(*channels)
    return _s(lib().ref_gen_cnn(batch, image_hw[0], image_hw[1], arr, len(channels),
                                filter_hw[0], filter_hw[1], int(backward), dtype_bytes))


def assignment(graph_json: str, mode: str, k: int) -> dict:
    return json.loads(_s(lib().ref_assignment(_b(graph_json), _b(mode), k)))


def kcuts(graph_json: str, k: int) -> dict:
    return json.loads(_s(lib().ref_kcuts(_b(graph_json), k)))


def graph_cost(graph_json: str, mode: str, k: int) -> dict:
    return json.loads(_s(lib().ref_graph_cost(_b(graph_json), _b(mode), k)))


def flat_hierarchy(k: int, label="nvswitch", bw=9e11) -> str:
    if k == 0:
        return json.dumps({"levels": []})
    return json.dumps({"levels": [{"label": label, "fanout": 1 << k, "bandwidth_bytes_per_s": bw}]})


def plan(graph_json: str, mode: str, k: int, hierarchy_json: str | None = None) -> str:
    h = hierarchy_json if hierarchy_json is not None else flat_hierarchy(k)
    return _s(lib().ref_plan(_b(graph_json), _b(mode), k, _b(h)))


def plan_roundtrip(plan_json: str) -> str:
    return _s(lib().ref_plan_roundtrip(_b(plan_json)))


def simulate_traffic(plan_json: str, hierarchy_json: str = "") -> dict:
    return json.loads(_s(lib().ref_simulate_traffic(_b(plan_json), _b(hierarchy_json))))


def execute_numeric(plan_json: str, seed: int) -> dict:
    a, r, s = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    v = ctypes.c_int64()
    if lib().ref_execute_numeric(_b(plan_json), seed, ctypes.byref(a), ctypes.byref(r),
                                 ctypes.byref(v), ctypes.byref(s)):
        raise RefError(lib().ref_last_error().decode())
    return {"max_abs": a.value, "max_rel": r.value, "values": v.value, "seed": seed,
            "seconds": s.value}


def execute_numeric_parallel(plan_json: str, seed: int, threads: int) -> float:
    s = ctypes.c_double()
    if lib().ref_execute_numeric_parallel(_b(plan_json), seed, threads, ctypes.byref(s)):
        raise RefError(lib().ref_last_error().decode())
    return s.value


def serial_seconds(plan_json: str, seed: int) -> float:
    s = ctypes.c_double()
    if lib().ref_serial_seconds(_b(plan_json), seed, ctypes.byref(s)):
        raise RefError(lib().ref_last_error().decode())
    return s.value


class Session:
    """execute_numeric's node loop, keeping every node value (fp64) for golden data."""

    def __init__(self, plan_json: str, seed: int):
        self.plan = json.loads(plan_json)
        self._h = lib().ref_session_new(_b(plan_json), seed)
        if not self._h:
            raise RefError(lib().ref_last_error().decode())
        self._nodes = {n["id"]: n for n in self.plan["nodes"]}
        self._shapes = {t["id"]: t["shape"] for t in self.plan["graph"]["tensors"]}

    def close(self):
        if self._h:
            lib().ref_session_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def times(self):
        a, b = ctypes.c_double(), ctypes.c_double()
        lib().ref_session_times(self._h, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def serial(self, tensor: str) -> np.ndarray:
        shape = self._shapes[tensor]
        out = np.empty(shape, dtype=np.float64)
        if lib().ref_session_serial(self._h, _b(tensor), out.ctypes.data_as(
                ctypes.POINTER(ctypes.c_double)), out.size):
            raise RefError(lib().ref_last_error().decode())
        return out

    def node(self, node_id: str) -> np.ndarray:
        reg = self._nodes[node_id]["region"]
        out = np.empty([hi - lo for lo, hi in reg], dtype=np.float64)
        if lib().ref_session_node(self._h, _b(node_id), out.ctypes.data_as(
                ctypes.POINTER(ctypes.c_double)), out.size):
            raise RefError(lib().ref_last_error().decode())
        return out


class Pool:
    """`threads` independent copies of the reference's tiled node loop on the same plan;
    step() runs all copies concurrently (one per host thread) and returns the wall time."""

    def __init__(self, plan_json: str, seed: int, threads: int):
        self.threads = threads
        self._h = lib().ref_pool_new(_b(plan_json), seed, threads)
        if not self._h:
            raise RefError(lib().ref_last_error().decode())

    def step(self) -> float:
        s = ctypes.c_double()
        if lib().ref_pool_step(self._h, ctypes.byref(s)):
            raise RefError(lib().ref_last_error().decode())
        return s.value

    def close(self):
        if self._h:
            lib().ref_pool_free(self._h)
            self._h = None

    def __del__(self):
        self.close()
