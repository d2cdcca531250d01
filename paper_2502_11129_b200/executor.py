"""Executor boundary — Python mirror of hetbench's batch contract
(/root/reference/proj/include/hetbench/executor.hpp:17-128) over the C ABI.

``GpuExecutor`` is the B200 back-end that takes the accelerator slot
(``synthetic_executor``, src/executor.cpp:137-170): ``run(BatchRequest)``
returns a ``BatchResult`` whose results are bit-identical to the reference
``simulate`` (src/simkernel.cpp:187-203) seed for seed, or raises
``BatchFailure`` carrying the failed seeds (sorted) and the completed results,
with the reference's message format (executor.cpp:20-28).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import RESULT_DTYPE, lib

KSIM_DT = 0.002


class ModelKind(enum.IntEnum):
    """hetbench::ModelKind (simkernel.hpp:14), same ordinals; CpgHinge (4) is
    the CPG / hinge modular robot of BASELINE config 3, which the reference
    does not have — defined by oracle/hb_oracle.c, parity
    against that definition only."""
    Box = 0
    BoxAndBall = 1
    ArmWithRope = 2
    Humanoid = 3
    CpgHinge = 4


_NAMES = ("box", "box_and_ball", "arm_with_rope", "humanoid", "cpg_hinge")
REFERENCE_MODELS = (ModelKind.Box, ModelKind.BoxAndBall, ModelKind.ArmWithRope, ModelKind.Humanoid)
ALL_MODELS = tuple(ModelKind)


def to_string(kind: ModelKind) -> str:
    return _NAMES[int(kind)]


def parse_model_kind(name: str) -> ModelKind:
    """simkernel.cpp:52-56."""
    for k in ModelKind:
        if _NAMES[int(k)] == name:
            return k
    raise ValueError(f"unknown model kind: {name}")


def body_count(kind: ModelKind) -> int:
    return int(lib.hb_body_count(int(kind)))


def constraint_count(kind: ModelKind) -> int:
    return int(lib.hb_constraint_count(int(kind)))


def state_rows(kind: ModelKind) -> int:
    return int(lib.hb_state_rows(int(kind)))


class NumericalBlowup(RuntimeError):
    """hetbench::numerical_blowup (simkernel.hpp:62-65)."""


class BatchFailure(RuntimeError):
    """hetbench::batch_failure (executor.hpp:34-45): failed = [(seed, message)]
    sorted, completed = results of the variants that finished, in order."""

    def __init__(self, failed, completed):
        self.failed = sorted(failed)
        self.completed = completed
        first_seed, first_msg = self.failed[0]
        msg = f"batch failed for seed {first_seed}"
        if len(self.failed) > 1:
            msg += f" (+{len(self.failed) - 1} more)"
        msg += ": " + first_msg
        super().__init__(msg)


@dataclass
class BatchRequest:
    kind: ModelKind = ModelKind.Box
    seeds: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))
    steps: int = 1

    def __post_init__(self):
        self.kind = ModelKind(self.kind)
        self.seeds = np.ascontiguousarray(np.asarray(self.seeds, dtype=np.uint64))


@dataclass
class BatchResult:
    """results: structured array (seed, fitness, checksum, steps_executed),
    request order — the 32-byte VariantResult layout."""
    results: np.ndarray
    wall_time_s: float = 0.0
    utilization_trace: list = field(default_factory=list)


def validate_request(request: BatchRequest) -> None:
    """executor.cpp:60-65."""
    if len(request.seeds) == 0:
        raise ValueError("batch request: seeds must be non-empty")
    if request.steps < 1:
        raise ValueError("batch request: steps must be >= 1")


def format_blowup(seed: int, fail_step: int, dt: float = KSIM_DT) -> str:
    buf = C.create_string_buffer(256)
    lib.hb_format_blowup(int(seed), int(fail_step), dt, buf, 256)
    return buf.value.decode()


def _raise_partial(seeds: np.ndarray, out: np.ndarray, fail: np.ndarray):
    bad = np.nonzero(fail)[0]
    failed = [(int(seeds[i]), format_blowup(int(seeds[i]), int(fail[i]))) for i in bad]
    completed = out[fail == 0].copy()
    raise BatchFailure(failed, completed)


class BatchExecutor:
    """hetbench::batch_executor (executor.hpp:68-73)."""

    def run(self, request: BatchRequest) -> BatchResult:  # pragma: no cover - interface
        raise NotImplementedError

    def name(self) -> str:  # pragma: no cover - interface
        raise NotImplementedError


class DeviceContext:
    """Owns one hb_ctx (one device, one stream, pinned + device buffers)."""

    def __init__(self, device: int = 0, host_threads: int = 0):
        h = C.c_void_p()
        st = lib.hb_ctx_create(device, C.byref(h))
        if st != _lib.HB_OK:
            raise RuntimeError(f"hb_ctx_create({device}) failed [{st}]: {_lib.global_error()}")
        self.handle = h.value
        self.device = device
        if host_threads:
            lib.hb_ctx_set_host_threads(self.handle, host_threads)

    def error(self) -> str:
        return (lib.hb_last_error(self.handle) or b"").decode()

    def check(self, st: int, what: str) -> None:
        if st == _lib.HB_INVALID_ARG:
            raise ValueError(self.error())
        if st not in (_lib.HB_OK, _lib.HB_BLOWUP_PARTIAL):
            raise RuntimeError(f"{what} failed [{st}]: {self.error()}")

    @property
    def stream(self) -> int:
        return int(lib.hb_ctx_stream(self.handle) or 0)

    def close(self):
        if getattr(self, "handle", None):
            lib.hb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- staged (device-resident) path, used by bench.py for kernel timing
    def stage(self, kind: ModelKind, seeds: np.ndarray) -> None:
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        self._staged = seeds
        self.check(lib.hb_stage(self.handle, int(kind), _lib.ptr(seeds), len(seeds)), "hb_stage")

    def launch(self, steps: int) -> None:
        self.check(lib.hb_launch(self.handle, steps), "hb_launch")

    def synchronize(self) -> None:
        self.check(lib.hb_synchronize(self.handle), "hb_synchronize")

    def fetch(self):
        n = len(self._staged)
        out = np.zeros(n, dtype=RESULT_DTYPE)
        fail = np.zeros(n, dtype=np.uint64)
        self.check(lib.hb_fetch(self.handle, _lib.ptr(out), _lib.ptr(fail)), "hb_fetch")
        return out, fail

    def last_launch_stats(self):
        """(failed variants, exact step replays) of the last fetched batch."""
        f, r = C.c_uint64(0), C.c_uint64(0)
        self.check(lib.hb_last_launch_stats(self.handle, C.byref(f), C.byref(r)), "stats")
        return int(f.value), int(r.value)

    def set_zero_copy(self, enable: bool) -> None:
        """Box zero-copy path for pinned seeds + results (default on)."""
        self.check(lib.hb_ctx_set_zero_copy(self.handle, int(bool(enable))), "hb_ctx_set_zero_copy")

    def work_counter(self) -> int:
        """Running total of algorithmic FP64 ops executed by Box launches
        (hb_work_counter; 16 per variant-step, 10 at the grounded fixed point)."""
        v = C.c_uint64(0)
        self.check(lib.hb_work_counter(self.handle, C.byref(v)), "hb_work_counter")
        return int(v.value)

    def calibrate(self, kind: ModelKind, steps: int, probe_n: int, repeats: int = 5):
        """hb_calibrate on this context: (median per-launch seconds of the
        probe, relative spread); raises if the device fails the probe."""
        t = np.zeros(1)
        sp = np.zeros(1)
        ok = np.zeros(1, dtype=np.int32)
        handles = (C.c_void_p * 1)(self.handle)
        st = lib.hb_calibrate(C.cast(handles, C.c_void_p), 1, int(kind), int(probe_n), int(steps),
                              int(repeats), _lib.ptr(t), _lib.ptr(sp), _lib.ptr(ok))
        if st != _lib.HB_OK or not ok[0]:
            raise RuntimeError(f"calibrate failed [{st}]: {self.error() or _lib.global_error()}")
        return float(t[0]), float(sp[0])

    def inject_fault(self, mode: int, seed: int = 0) -> None:
        """Test seam (hb_ctx_inject_fault): HB_FAULT_BLOWUP reports the variants
        with this seed as blown up at step 1; HB_FAULT_DEVICE makes every
        hb_run_batch fail as a dead device; HB_FAULT_NONE resets."""
        self.check(lib.hb_ctx_inject_fault(self.handle, int(mode), int(seed)), "hb_ctx_inject_fault")

    def set_precision(self, precision: int) -> None:
        """_lib.HB_PRECISION_FP64 (bit-exact product path, default) or
        _lib.HB_PRECISION_FP32 (throughput mode: float-float
        positions, FP32 increments; fitness within 1e-4 relative, not bit-exact)."""
        self.check(lib.hb_ctx_set_precision(self.handle, int(precision)), "hb_ctx_set_precision")

    def set_kernel(self, variant: int) -> None:
        """_lib.HB_KERNEL_AUTO (optimised) or _lib.HB_KERNEL_GENERIC (reference-order cross-check)."""
        self.check(lib.hb_ctx_set_kernel(self.handle, int(variant)), "hb_ctx_set_kernel")

    def check_fast_math(self, x: np.ndarray, y: np.ndarray):
        """(sqrt_mismatch, div_mismatch, sqrt_flagged, div_flagged) of the
        kernels' branch-free sqrt / div replicas against the library on the device."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        r = [C.c_uint64(0) for _ in range(4)]
        self.check(lib.hb_check_fast_math(self.handle, _lib.ptr(x), _lib.ptr(y), len(x),
                                          *[C.byref(v) for v in r]), "hb_check_fast_math")
        return tuple(int(v.value) for v in r)

    def fp64_peak(self):
        ops = C.c_double(0)
        ms = C.c_double(0)
        self.check(lib.hb_fp64_peak(self.handle, C.byref(ops), C.byref(ms)), "hb_fp64_peak")
        return ops.value, ms.value


class GpuExecutor(BatchExecutor):
    """The B200 accelerator back-end: one device, one persistent kernel per batch."""

    def __init__(self, device: int = 0, host_threads: int = 0, kernel: int = _lib.HB_KERNEL_AUTO,
                 monitor: bool = False, precision: int = _lib.HB_PRECISION_FP64):
        self.ctx = DeviceContext(device, host_threads)
        # utilisation trace (hb_ctx_set_monitor: NVML at 20 Hz + the call's
        # kernel-busy share), like cpu_executor(monitor=true)
        self.monitor = monitor
        if monitor:
            self.ctx.check(lib.hb_ctx_set_monitor(self.ctx.handle, 1), "hb_ctx_set_monitor")
        if kernel != _lib.HB_KERNEL_AUTO:
            self.ctx.set_kernel(kernel)
        if precision != _lib.HB_PRECISION_FP64:
            self.ctx.set_precision(precision)

    def name(self) -> str:
        return "accel"

    def reserve(self, kind: ModelKind, n: int) -> None:
        """Size the context's buffers for batches of up to n variants of kind
        and load their kernel (hb_ctx_reserve): start-up work a single-probe
        calibrate would otherwise time as accelerator speed."""
        self.ctx.check(lib.hb_ctx_reserve(self.ctx.handle, int(kind), int(n)), "hb_ctx_reserve")

    def utilization_trace(self):
        """[(t_s, accel_percent)] of the last monitored call (hb_last_utilization)."""
        n = C.c_size_t(0)
        lib.hb_last_utilization(self.ctx.handle, None, 0, C.byref(n))
        buf = np.zeros(2 * n.value)
        lib.hb_last_utilization(self.ctx.handle, _lib.ptr(buf), n.value, C.byref(n))
        return [(float(buf[2 * i]), float(buf[2 * i + 1])) for i in range(n.value)]

    def run_raw(self, kind: ModelKind, seeds: np.ndarray, steps: int):
        """(results, fail_step or None, wall_s, status) without raising on
        blow-up; fail_step is only materialised when something blew up."""
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        n = len(seeds)
        out = _lib.pinned.empty(n, RESULT_DTYPE)
        wall = C.c_double(0)
        st = lib.hb_run_batch(self.ctx.handle, int(kind), _lib.ptr(seeds), n, int(steps),
                              _lib.ptr(out), None, C.byref(wall))
        self.ctx.check(st, "hb_run_batch")
        fail = None  # per-variant failure steps only exist after a blow-up
        if st == _lib.HB_BLOWUP_PARTIAL:
            fail = np.zeros(n, dtype=np.uint64)
            self.ctx.check(lib.hb_last_fail_steps(self.ctx.handle, _lib.ptr(fail), n), "fail steps")
        return out, fail, wall.value, st

    def run(self, request: BatchRequest) -> BatchResult:
        validate_request(request)
        out, fail, wall, st = self.run_raw(request.kind, request.seeds, request.steps)
        trace = self.utilization_trace() if self.monitor else []
        if st == _lib.HB_BLOWUP_PARTIAL:
            _raise_partial(request.seeds, out, fail)
        return BatchResult(out, wall, trace)

    def run_states(self, kind: ModelKind, pos: np.ndarray, vel: np.ndarray, rest: np.ndarray,
                   steps: int = 1, dt: float = KSIM_DT, seeds=None, cpg=None):
        """Run from explicit initial states (known-answer tests).  pos/vel:
        (N, n, 3); rest: (N, m); cpg (CpgHinge only): (N, 16) = x[4], y[4],
        omega[4], coupling[4].  Returns (results, fail_step, pos, vel)."""
        pos = np.asarray(pos, dtype=np.float64)
        vel = np.asarray(vel, dtype=np.float64)
        N, nb = pos.shape[0], pos.shape[1]
        m = constraint_count(kind)
        rest = np.asarray(rest, dtype=np.float64).reshape(N, m)
        parts = [pos.reshape(N, 3 * nb).T, vel.reshape(N, 3 * nb).T, rest.T]
        if int(kind) == int(ModelKind.CpgHinge):
            parts.append(np.asarray(cpg, dtype=np.float64).reshape(N, 16).T)
        soa = np.concatenate(parts, axis=0)
        soa = np.ascontiguousarray(soa)
        final = np.empty_like(soa)
        out = np.empty(N, dtype=RESULT_DTYPE)
        fail = np.empty(N, dtype=np.uint64)
        sd = None if seeds is None else np.ascontiguousarray(seeds, dtype=np.uint64)
        st = lib.hb_run_states(self.ctx.handle, int(kind), _lib.ptr(soa), N, int(steps), float(dt),
                               None if sd is None else _lib.ptr(sd), _lib.ptr(out), _lib.ptr(fail),
                               _lib.ptr(final))
        self.ctx.check(st, "hb_run_states")
        fp = final[: 3 * nb].T.reshape(N, nb, 3)
        fv = final[3 * nb: 6 * nb].T.reshape(N, nb, 3)
        return out, fail, fp.copy(), fv.copy()


class MultiGpuExecutor(BatchExecutor):
    """One context + one host thread per device (hb_run_batch_multi); the batch
    is cut into contiguous per-device slices (scheduler.cpp:122-127) and
    merged in seed order.  ``shares`` come from the N-way splitter
    (scheduler.plan_allocation_n); None splits evenly."""

    def __init__(self, devices: Sequence[int], host_threads: int = 0):
        self.ctxs = [DeviceContext(d, host_threads) for d in devices]
        self.shares = None        # fixed per-device shares (sum = batch size), or
        self.device_times = None  # calibrated per-device probe times -> plan_allocation_n
        self.device_ok = None     # calibration's liveness flags (None = all alive)
        self.last_device_walls = None
        self.last_device_ok = None
        self.last_degraded = False

    def name(self) -> str:
        return f"accel x{len(self.ctxs)}"

    def run(self, request: BatchRequest) -> BatchResult:
        """hb_run_batch_multi: shares from ``shares``, else plan_allocation_n
        over ``device_times`` / ``device_ok`` (calibrate()), else even.  A
        device that fails is dropped and its slice re-planned over the
        survivors (``last_degraded``, ``last_device_ok``)."""
        validate_request(request)
        seeds = np.ascontiguousarray(request.seeds, dtype=np.uint64)
        n = len(seeds)
        cnt = len(self.ctxs)
        handles = (C.c_void_p * cnt)(*[c.handle for c in self.ctxs])
        sh = None
        if self.shares is not None:
            sh = np.ascontiguousarray(self.shares, dtype=np.uint64)
        elif self.device_times is not None:
            from .scheduler import plan_allocation_n
            sh = np.ascontiguousarray(plan_allocation_n(self.device_times, n, self.device_ok), dtype=np.uint64)
        out = np.empty(n, dtype=RESULT_DTYPE)
        fail = np.empty(n, dtype=np.uint64)
        walls = np.zeros(cnt)
        wall = C.c_double(0)
        dok = np.zeros(cnt, dtype=np.int32)
        degraded = C.c_int(0)
        st = lib.hb_run_batch_multi(C.cast(handles, C.c_void_p), cnt,
                                    None if sh is None else _lib.ptr(sh), int(request.kind),
                                    _lib.ptr(seeds), n, int(request.steps), _lib.ptr(out),
                                    _lib.ptr(fail), _lib.ptr(walls), C.byref(wall),
                                    _lib.ptr(dok), C.byref(degraded))
        if st == _lib.HB_INVALID_ARG:
            raise ValueError(_lib.global_error())
        if st not in (_lib.HB_OK, _lib.HB_BLOWUP_PARTIAL):
            raise RuntimeError(f"hb_run_batch_multi failed [{st}]: {_lib.global_error()}")
        self.last_device_walls = walls
        self.last_device_ok = [bool(x) for x in dok]
        self.last_degraded = bool(degraded.value)
        if st == _lib.HB_BLOWUP_PARTIAL:
            _raise_partial(seeds, out, fail)
        return BatchResult(out, wall.value, [])

    def calibrate(self, kind: ModelKind, steps: int, probe_n: int, repeats: int = 5,
                  snap_tol: float = 0.01):
        """The paper's calibrate step on every device at once (hb_calibrate:
        a >= 5 ms probe timed with CUDA events, median of `repeats`), then
        hb_snap_equal_times (equal devices -> equal shares).  Sets and returns
        (device_times, device_ok, spreads)."""
        cnt = len(self.ctxs)
        handles = (C.c_void_p * cnt)(*[c.handle for c in self.ctxs])
        t = np.zeros(cnt)
        sp = np.zeros(cnt)
        ok = np.zeros(cnt, dtype=np.int32)
        st = lib.hb_calibrate(C.cast(handles, C.c_void_p), cnt, int(kind), int(probe_n), int(steps),
                              int(repeats), _lib.ptr(t), _lib.ptr(sp), _lib.ptr(ok))
        if st == _lib.HB_INVALID_ARG:
            raise ValueError(_lib.global_error())
        if st != _lib.HB_OK:
            raise RuntimeError(_lib.global_error())
        snapped = np.zeros(cnt)
        lib.hb_snap_equal_times(_lib.ptr(t), _lib.ptr(sp), _lib.ptr(ok), cnt, float(snap_tol),
                                _lib.ptr(snapped))
        self.device_times = [float(x) for x in snapped]
        self.device_ok = [bool(x) for x in ok]
        self.shares = None
        return self.device_times, self.device_ok, [float(x) for x in sp]


def build_states(kind: ModelKind, seeds) -> np.ndarray:
    """Host initialiser output (SoA rows x N) — build_model for each seed."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    rows = state_rows(kind)
    soa = np.empty((rows, len(seeds)))
    st = lib.hb_build_states(int(kind), _lib.ptr(seeds), len(seeds), _lib.ptr(soa), len(seeds))
    if st != _lib.HB_OK:
        raise ValueError(_lib.global_error())
    return soa


def pinned_seeds(seeds) -> np.ndarray:
    """A copy of `seeds` in mapped page-locked memory (recycled pool): H2D
    without staging, and the Box zero-copy path."""
    src = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = _lib.pinned.empty(len(src), np.uint64)
    out[:] = src
    return out


def kernel_name(kind: ModelKind, n: int) -> str:
    buf = C.create_string_buffer(128)
    lib.hb_kernel_name(int(kind), n, buf, 128)
    return buf.value.decode()


def device_count() -> int:
    return int(lib.hb_device_count())
