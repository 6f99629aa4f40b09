"""ctypes binding of libzk_b200.so (the C ABI in include/zk_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2409_19156_b200/csrc``). There is no CPU fallback: if the
library is missing this module raises ImportError at import time, and every
compute entry point raises RuntimeError when no CUDA device is usable.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint32, c_void_p

import numpy as np

LIB_PATH = os.environ.get("ZK_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libzk_b200.so")

ZK_OK = 0
ZK_EINVAL = -1
ZK_ECUDA = -2
ZK_ENOMEM = -3
ZK_ENODEV = -4

ZK_HOST_INPUT = 1
ZK_HOST_OUTPUT = 2
ZK_ASYNC = 4
ZK_STORE_SCALAR = 8

CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "or `make -C paper_2409_19156_b200/csrc` (there is no CPU fallback)"
    )

lib = ctypes.CDLL(LIB_PATH)

_i32p = POINTER(c_int32)
_i64p = POINTER(c_int64)
_dp = POINTER(c_double)

# name -> (restype, argtypes); kept in sync with include/zk_b200.h
SIGNATURES = {
    "zk_last_error": (ctypes.c_char_p, []),
    "zk_version": (c_int, []),
    "zk_device_count": (c_int, [POINTER(c_int)]),
    "zk_ctx_create": (c_int, [c_int, POINTER(c_void_p)]),
    "zk_ctx_destroy": (c_int, [c_void_p]),
    "zk_ctx_set_stream": (c_int, [c_void_p, c_void_p]),
    "zk_ctx_synchronize": (c_int, [c_void_p]),
    "zk_ctx_release_buffers": (c_int, [c_void_p]),
    "zk_ctx_launch_count": (c_int, [c_void_p, _i64p]),
    "zk_host_register": (c_int, [c_void_p, ctypes.c_size_t]),
    "zk_host_unregister": (c_int, [c_void_p]),
    "zk_plan_describe": (c_int, [_i32p, _i32p, c_int64, _i32p, _i32p, _i32p, _i64p]),
    "zk_step_counters": (c_int, [_i32p, _i32p, c_int64, c_int, c_int, _i64p, _i64p]),
    "zk_plan_create": (c_int, [c_void_p, _i32p, _i32p, c_int64, c_int, POINTER(c_void_p)]),
    "zk_plan_destroy": (c_int, [c_void_p]),
    "zk_plan_info": (c_int, [c_void_p, _i64p, _i64p, _i64p, _i64p]),
    "zk_radial_eval": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int,
                               c_void_p, c_int64, c_int64, c_uint32]),
    "zk_zernike_eval": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                                c_int, c_void_p, c_int64, c_int64, c_uint32]),
    "zk_series_eval": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                               c_void_p, c_int64, c_int64, c_void_p, c_int64, c_uint32]),
    "zk_gram_accumulate": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                   c_void_p, c_void_p, c_void_p, c_uint32]),
    "zk_jacobi_chain": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int,
                                c_void_p, c_int64, c_uint32]),
    "zk_direct_eval": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                               c_int64, c_void_p, c_int64, c_uint32]),
    "zk_ztt_eval": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                            c_void_p, c_int64, c_uint32]),
    "zk_radial_eval_dd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int,
                                  c_void_p, c_int64, c_uint32]),
    "zk_gram_packed_count": (c_int64, [c_int64]),
    "zk_gram_pack": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_uint32]),
    "zk_gram_unpack": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_uint32]),
    "zk_nccl_version": (c_int, [POINTER(c_int)]),
    "zk_gram_allreduce": (c_int, [POINTER(c_void_p), c_int, POINTER(c_void_p), POINTER(c_void_p),
                                  c_int64, c_uint32]),
    "zk_comm_unique_id": (c_int, [c_void_p]),
    "zk_comm_create": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(c_void_p)]),
    "zk_comm_info": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int)]),
    "zk_comm_destroy": (c_int, [c_void_p]),
    "zk_gram_allreduce_comm": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_uint32]),
    "zk_emul_colexp": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "zk_emul_slices": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int, c_void_p,
                               c_int64, c_int64, c_int64, c_void_p]),
    "zk_emul_accumulate": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int, c_int,
                                   c_void_p, c_int64, c_void_p]),
    "zk_host_alloc": (c_int, [c_int64, POINTER(c_void_p)]),
    "zk_host_free": (c_int, [c_void_p]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)  # AttributeError here = library/header mismatch
    _fn.restype = _res
    _fn.argtypes = _args


class ZKError(RuntimeError):
    """A CUDA-side failure reported by libzk_b200."""


def check(rc: int, what: str) -> None:
    if rc == ZK_OK:
        return
    msg = lib.zk_last_error().decode(errors="replace")
    if rc == ZK_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise ZKError(f"{what} failed ({rc}): {msg}")


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def ptr_i32(a: np.ndarray):
    return a.ctypes.data_as(_i32p)


# --------------------------------------------------------------------------
# host-only planner (usable without a GPU)
# --------------------------------------------------------------------------

def describe(mode_n: np.ndarray, mode_m: np.ndarray):
    """(unique_n, unique_m, scatter) -- zk/modes.py:108-125 semantics."""
    n, m = i32(mode_n), i32(mode_m)
    M = n.size
    un = np.empty(max(M, 1), np.int32)
    um = np.empty(max(M, 1), np.int32)
    sc = np.empty(max(M, 1), np.int32)
    U = c_int64(0)
    check(lib.zk_plan_describe(ptr_i32(n), ptr_i32(m), M, ptr_i32(un), ptr_i32(um),
                               ptr_i32(sc), ctypes.byref(U)), "zk_plan_describe")
    return un[: U.value].copy(), um[: U.value].copy(), sc[:M].copy()


def step_counters(mode_n, mode_m, deriv_order: int, shared: bool) -> tuple[int, int]:
    n, m = i32(mode_n), i32(mode_m)
    steps, chains = c_int64(0), c_int64(0)
    check(lib.zk_step_counters(ptr_i32(n), ptr_i32(m), n.size, int(deriv_order), int(shared),
                               ctypes.byref(steps), ctypes.byref(chains)), "zk_step_counters")
    return steps.value, chains.value


# --------------------------------------------------------------------------
# contexts and plans
# --------------------------------------------------------------------------

class Context:
    """One zk_ctx (CUDA stream + scratch) on one device."""

    def __init__(self, device: int = 0):
        h = c_void_p()
        check(lib.zk_ctx_create(int(device), ctypes.byref(h)), f"zk_ctx_create(device={device})")
        self.handle = h
        self.device = int(device)
        self.lock = threading.Lock()

    def launches(self) -> int:
        c = c_int64(0)
        check(lib.zk_ctx_launch_count(self.handle, ctypes.byref(c)), "zk_ctx_launch_count")
        return c.value

    def release_buffers(self) -> None:
        """Free the context's cached scratch and pinned bounce buffers."""
        check(lib.zk_ctx_release_buffers(self.handle), "zk_ctx_release_buffers")

    def set_stream(self, stream_ptr: int | None) -> None:
        """Launch on the caller's cudaStream_t; None / 0 = the ctx's own stream."""
        check(lib.zk_ctx_set_stream(self.handle, c_void_p(stream_ptr or 0)), "zk_ctx_set_stream")

    def use_torch_stream(self, device: int | None = None) -> None:
        """Launch on torch's current stream of this ctx's device. torch's
        default stream is the legacy default stream (handle 0), which the C
        ABI would read as "the ctx's own (non-blocking) stream"; it is passed
        as cudaStreamLegacy instead, so the kernels stay ordered with torch's
        work either way."""
        import torch
        h = torch.cuda.current_stream(self.device if device is None else device).cuda_stream
        self.set_stream(h if h else CUDA_STREAM_LEGACY)

    def synchronize(self) -> None:
        check(lib.zk_ctx_synchronize(self.handle), "zk_ctx_synchronize")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and lib is not None:
            lib.zk_ctx_destroy(h)
            self.handle = None


class Plan:
    """zk_plan: alpha groups + exact coefficients for one mode list, on device."""

    def __init__(self, ctx: Context, mode_n, mode_m, max_order: int = 3):
        self.ctx = ctx
        n, m = i32(mode_n), i32(mode_m)
        h = c_void_p()
        check(lib.zk_plan_create(ctx.handle, ptr_i32(n), ptr_i32(m), n.size, int(max_order),
                                 ctypes.byref(h)), "zk_plan_create")
        self.handle = h
        self.M = int(n.size)
        self.max_order = int(max_order)

    def info(self) -> dict:
        M, U, G, N = c_int64(), c_int64(), c_int64(), c_int64()
        check(lib.zk_plan_info(self.handle, ctypes.byref(M), ctypes.byref(U), ctypes.byref(G),
                               ctypes.byref(N)), "zk_plan_info")
        return {"M": M.value, "U": U.value, "groups": G.value, "max_n": N.value}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and lib is not None:
            lib.zk_plan_destroy(h)
            self.handle = None


class Comm:
    """zk_comm: one NCCL rank of the K5 normal-equation allreduce, bound to a
    Context (one process per GPU). ``unique_id()`` on rank 0, shared by the
    launcher (e.g. a torch.distributed broadcast), then ``Comm(ctx, id, N, r)``
    on every rank."""

    def __init__(self, ctx: Context, uid: bytes, nranks: int, rank: int):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.ctx = ctx
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        h = c_void_p()
        check(lib.zk_comm_create(ctx.handle, buf, int(nranks), int(rank), ctypes.byref(h)),
              "zk_comm_create")
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib.zk_comm_unique_id(buf), "zk_comm_unique_id")
        return buf.raw

    def info(self) -> tuple[int, int]:
        n, r = c_int(0), c_int(0)
        check(lib.zk_comm_info(self.handle, ctypes.byref(n), ctypes.byref(r)), "zk_comm_info")
        return n.value, r.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and lib is not None:
            lib.zk_comm_destroy(h)
            self.handle = None


def nccl_version() -> int:
    v = c_int(0)
    check(lib.zk_nccl_version(ctypes.byref(v)), "zk_nccl_version")
    return v.value


_ctx_lock = threading.Lock()
_contexts: dict[int, Context] = {}
_plans: dict = {}
_PLAN_CACHE = 16


def context(device: int | None = None) -> Context:
    """Process-wide context for ``device`` (default: ZK_DEVICE env or 0)."""
    if device is None:
        device = int(os.environ.get("ZK_DEVICE", "0"))
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def plan_for(ctx: Context, mode_n: np.ndarray, mode_m: np.ndarray) -> Plan:
    """Cached device plan for this exact column list (all orders 0..3)."""
    n, m = i32(mode_n), i32(mode_m)
    key = (ctx.device, n.tobytes(), m.tobytes())
    with _ctx_lock:
        p = _plans.get(key)
        if p is not None:
            _plans[key] = _plans.pop(key)  # LRU refresh
            return p
    p = Plan(ctx, n, m, 3)
    with _ctx_lock:
        _plans[key] = p
        while len(_plans) > _PLAN_CACHE:
            _plans.pop(next(iter(_plans)))
    return p


def dptr(a: np.ndarray) -> int:
    return a.ctypes.data
