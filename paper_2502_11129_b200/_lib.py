"""ctypes binding of the C ABI in include/hbgpu.h (libhbgpu.so, built in-tree).

The product has no CPU fallback: if the shared library is missing this module
raises at import time, and a context cannot be created without an sm_100
device (HB_NO_DEVICE).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libhbgpu.so")

HB_OK, HB_INVALID_ARG, HB_CUDA_ERROR, HB_BLOWUP_PARTIAL, HB_NO_DEVICE = range(5)

RESULT_DTYPE = np.dtype([("seed", "<u8"), ("fitness", "<f8"), ("checksum", "<u8"),
                         ("steps_executed", "<u8")])

# Every symbol include/hbgpu.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "hb_abi_version", "hb_device_count", "hb_body_count", "hb_constraint_count",
    "hb_state_rows", "hb_global_error", "hb_ctx_create", "hb_ctx_destroy", "hb_last_error",
    "hb_ctx_device", "hb_ctx_stream", "hb_ctx_set_host_threads", "hb_run_batch",
    "hb_build_states", "hb_run_states", "hb_stage", "hb_launch", "hb_synchronize", "hb_fetch",
    "hb_kernel_name", "hb_format_blowup", "hb_plan_allocation", "hb_plan_allocation_n",
    "hb_run_batch_multi", "hb_fp64_peak", "hb_ctx_set_kernel", "hb_check_fast_math",
    "hb_last_launch_stats", "hb_run_ea", "hb_eval_device", "hb_ea_init_genomes",
    "hb_ea_select_vary", "hb_host_alloc", "hb_host_free", "hb_last_fail_steps",
    "hb_ctx_set_zero_copy", "hb_ctx_set_precision", "hb_work_counter", "hb_ctx_inject_fault",
    "hb_calibrate", "hb_snap_equal_times", "hb_ctx_set_monitor", "hb_last_utilization", "hb_ctx_reserve",
)

HB_KERNEL_AUTO, HB_KERNEL_GENERIC = 0, 1
HB_PRECISION_FP64, HB_PRECISION_FP32 = 0, 1
HB_FAULT_NONE, HB_FAULT_BLOWUP, HB_FAULT_DEVICE = 0, 1, 2


class PhaseProfile(C.Structure):
    _fields_ = [("selection_s", C.c_double), ("variation_s", C.c_double),
                ("evaluation_s", C.c_double), ("bookkeeping_s", C.c_double),
                ("total_s", C.c_double), ("host_overhead_s", C.c_double)]


class Plan(C.Structure):
    _fields_ = [("n_total", C.c_uint64), ("n_cpu", C.c_uint64), ("n_accel", C.c_uint64),
                ("accel_fraction", C.c_double), ("requested_accel_fraction", C.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2502_11129_b200/csrc). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    u64, dbl, i32, sz, vp = C.c_uint64, C.c_double, C.c_int, C.c_size_t, C.c_void_p
    P = C.POINTER
    sig = {
        "hb_abi_version": (i32, []),
        "hb_device_count": (i32, []),
        "hb_body_count": (i32, [i32]),
        "hb_constraint_count": (i32, [i32]),
        "hb_state_rows": (i32, [i32]),
        "hb_global_error": (C.c_char_p, []),
        "hb_ctx_create": (i32, [i32, P(vp)]),
        "hb_ctx_destroy": (None, [vp]),
        "hb_last_error": (C.c_char_p, [vp]),
        "hb_ctx_device": (i32, [vp]),
        "hb_ctx_stream": (vp, [vp]),
        "hb_ctx_set_host_threads": (i32, [vp, i32]),
        "hb_run_batch": (i32, [vp, i32, vp, sz, u64, vp, vp, P(dbl)]),
        "hb_build_states": (i32, [i32, vp, sz, vp, sz]),
        "hb_run_states": (i32, [vp, i32, vp, sz, u64, dbl, vp, vp, vp, vp]),
        "hb_stage": (i32, [vp, i32, vp, sz]),
        "hb_launch": (i32, [vp, u64]),
        "hb_synchronize": (i32, [vp]),
        "hb_fetch": (i32, [vp, vp, vp]),
        "hb_kernel_name": (i32, [i32, sz, C.c_char_p, sz]),
        "hb_format_blowup": (i32, [u64, u64, dbl, C.c_char_p, sz]),
        "hb_plan_allocation": (i32, [dbl, dbl, i32, i32, u64, P(Plan)]),
        "hb_plan_allocation_n": (i32, [vp, vp, i32, u64, vp]),
        "hb_run_batch_multi": (i32, [vp, i32, vp, i32, vp, sz, u64, vp, vp, vp, P(dbl), vp, vp]),
        "hb_calibrate": (i32, [vp, i32, i32, u64, u64, i32, vp, vp, vp]),
        "hb_ctx_set_monitor": (i32, [vp, i32]),
        "hb_ctx_reserve": (i32, [vp, i32, sz]),
        "hb_last_utilization": (i32, [vp, vp, sz, P(sz)]),
        "hb_snap_equal_times": (i32, [vp, vp, vp, i32, dbl, vp]),
        "hb_fp64_peak": (i32, [vp, P(dbl), P(dbl)]),
        "hb_ctx_set_kernel": (i32, [vp, i32]),
        "hb_last_launch_stats": (i32, [vp, P(u64), P(u64)]),
        "hb_run_ea": (i32, [vp, i32, vp, i32, sz, u64, u64, u64, vp, vp, P(dbl), P(PhaseProfile),
                            vp, vp]),
        "hb_eval_device": (i32, [vp, i32, vp, sz, u64, vp, P(u64)]),
        "hb_ea_init_genomes": (i32, [vp, u64, sz, vp]),
        "hb_ea_select_vary": (i32, [vp, vp, vp, sz, u64, vp, vp]),
        "hb_host_alloc": (vp, [sz]),
        "hb_host_free": (None, [vp]),
        "hb_last_fail_steps": (i32, [vp, vp, sz]),
        "hb_ctx_set_zero_copy": (i32, [vp, i32]),
        "hb_ctx_set_precision": (i32, [vp, i32]),
        "hb_work_counter": (i32, [vp, P(u64)]),
        "hb_ctx_inject_fault": (i32, [vp, i32, u64]),
        "hb_check_fast_math": (i32, [vp, vp, vp, sz, P(u64), P(u64), P(u64), P(u64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


class PinnedPool:
    """Reusable page-locked result buffers.  Arrays handed out view pinned
    memory; when an array (and every view of it) is garbage-collected its
    buffer returns to the pool, so steady-state batches neither page-fault
    nor need a staging copy (the device DMAs straight into the array)."""

    def __init__(self):
        self._free = {}
        self._lock = threading.Lock()

    def empty(self, n: int, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = max(int(n) * dtype.itemsize, 1)
        cls = 1 << max(12, (nbytes - 1).bit_length())
        with self._lock:
            lst = self._free.get(cls)
            p = lst.pop() if lst else None
        if p is None:
            p = lib.hb_host_alloc(cls)
            if not p:
                return np.empty(n, dtype=dtype)  # not pinned: results go through staging
        raw = (C.c_char * cls).from_address(p)
        weakref.finalize(raw, self._release, cls, p)
        return np.frombuffer(raw, dtype=dtype, count=int(n))

    def _release(self, cls, p):
        with self._lock:
            self._free.setdefault(cls, []).append(p)


pinned = PinnedPool()


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def global_error() -> str:
    return (lib.hb_global_error() or b"").decode()
