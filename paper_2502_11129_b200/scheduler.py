"""Splitter — the paper's benchmark-driven allocator (§6) over the C ABI.

Mirrors /root/reference/proj/include/hetbench/scheduler.hpp:13-81:
``calibrate`` (scheduler.cpp:30-56), ``plan_allocation`` (:58-87, computed
natively by hb_plan_allocation, bit-for-bit), ``plan_allocation_optimal``
(:89-111), ``run_hybrid`` (:113-211), ``naive_sum``, ``format_plan``; plus
the N-way generalisation ``plan_allocation_n`` that shards one batch across
the GPUs of a box in proportion to measured per-GPU throughput and reduces to
``plan_allocation`` exactly for two back-ends.
"""
from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import lib
from .executor import (BatchExecutor, BatchRequest, BatchResult, ModelKind, validate_request)


@dataclass
class CalibrationProfile:
    kind: ModelKind = ModelKind.Box
    steps: int = 0
    probe_n: int = 0
    t_cpu_s: float = 0.0
    t_accel_s: float = 0.0
    ratio_accel_over_cpu: float = 0.0
    cpu_ok: bool = True
    accel_ok: bool = True


@dataclass
class AllocationPlan:
    n_total: int = 0
    n_cpu: int = 0
    n_accel: int = 0
    accel_fraction: float = 0.0
    requested_accel_fraction: float = 0.0


@dataclass
class HybridResult:
    wall_combined_s: float = 0.0
    t_cpu_part_s: float = 0.0
    t_accel_part_s: float = 0.0
    overhead_s: float = 0.0
    plan: AllocationPlan = field(default_factory=AllocationPlan)
    cpu_result: Optional[BatchResult] = None
    accel_result: Optional[BatchResult] = None
    merged: Optional[np.ndarray] = None
    degraded: bool = False


def _probe_request(kind, steps, probe_n) -> BatchRequest:
    return BatchRequest(kind, np.arange(probe_n, dtype=np.uint64), steps)


def calibrate(kind, steps, probe_n, cpu: BatchExecutor, accel: BatchExecutor) -> CalibrationProfile:
    """scheduler.cpp:30-56: probe seeds 0..probe_n-1 on each back-end,
    sequentially; a back-end that throws is flagged failed."""
    if probe_n < 1:
        raise ValueError("calibrate: probe_n must be >= 1")
    p = CalibrationProfile(ModelKind(kind), steps, probe_n)
    req = _probe_request(kind, steps, probe_n)
    try:
        p.t_cpu_s = cpu.run(req).wall_time_s
    except Exception:
        p.cpu_ok = False
    try:
        p.t_accel_s = accel.run(req).wall_time_s
    except Exception:
        p.accel_ok = False
    if not p.cpu_ok and not p.accel_ok:
        raise RuntimeError("calibrate: both back-ends failed")
    if p.cpu_ok and p.accel_ok:
        p.ratio_accel_over_cpu = p.t_accel_s / p.t_cpu_s
    return p


def snap_equal_times(times: Sequence[float], spreads: Optional[Sequence[float]] = None,
                     ok: Optional[Sequence[bool]] = None, min_rel_tol: float = 0.01) -> list[float]:
    """hb_snap_equal_times: if the alive back-ends' times agree within
    max(their largest measured relative spread, min_rel_tol), all of them get
    the mean time (equal shares) — measurement noise between identical GPUs
    must not turn into a permanent imbalance; otherwise unchanged."""
    cnt = len(times)
    t = np.ascontiguousarray(times, dtype=np.float64)
    sp = np.ascontiguousarray([0.0] * cnt if spreads is None else spreads, dtype=np.float64)
    okv = np.ascontiguousarray([1] * cnt if ok is None else [int(b) for b in ok], dtype=np.int32)
    out = np.zeros(cnt)
    lib.hb_snap_equal_times(_lib.ptr(t), _lib.ptr(sp), _lib.ptr(okv), cnt, float(min_rel_tol), _lib.ptr(out))
    return [float(x) for x in out]


def median_and_spread(samples: Sequence[float]) -> tuple[float, float]:
    """Median of the samples and their relative range (max - min) / median."""
    v = np.sort(np.asarray(samples, dtype=np.float64))
    med = float(np.median(v))
    return med, (float(v[-1] - v[0]) / med if med > 0 else 0.0)


def calibrate_n(kind, steps, probe_n, executors: Sequence[BatchExecutor], repeats: int = 5,
                snap_tol: Optional[float] = 0.01):
    """N-way calibration (scheduler.cpp:30-56 over N back-ends): the same
    probe on every back-end, sequentially, `repeats` times; a back-end's time
    is the median of its wall_time_s, and one that throws is flagged failed
    (time 0).  With snap_tol, times that agree within the measured spread
    snap to equal (snap_equal_times).  Returns (times, ok).  For GPU-only
    back-ends MultiGpuExecutor.calibrate times the probe with CUDA events on
    every device at once."""
    if probe_n < 1:
        raise ValueError("calibrate: probe_n must be >= 1")
    req = _probe_request(kind, steps, probe_n)
    times, ok, spreads = [], [], []
    for ex in executors:
        try:
            med, sp = median_and_spread([ex.run(req).wall_time_s for _ in range(max(1, repeats))])
            times.append(med)
            spreads.append(sp)
            ok.append(True)
        except Exception:  # noqa: BLE001 - a throwing back-end is dead (scheduler.cpp:40-49)
            times.append(0.0)
            spreads.append(0.0)
            ok.append(False)
    if not any(ok):
        raise RuntimeError("calibrate: all back-ends failed")
    if snap_tol is not None:
        times = snap_equal_times(times, spreads, ok, snap_tol)
    return times, ok


def plan_allocation(profile: CalibrationProfile, n_total: int) -> AllocationPlan:
    """Reverse-ratio split (scheduler.cpp:58-87), computed by hb_plan_allocation."""
    out = _lib.Plan()
    st = lib.hb_plan_allocation(float(profile.t_cpu_s), float(profile.t_accel_s),
                                int(profile.cpu_ok), int(profile.accel_ok), int(n_total),
                                C.byref(out))
    if st != _lib.HB_OK:
        raise ValueError(_lib.global_error())
    return AllocationPlan(out.n_total, out.n_cpu, out.n_accel, out.accel_fraction,
                          out.requested_accel_fraction)


def plan_allocation_n(times: Sequence[float], n_total: int,
                      ok: Optional[Sequence[bool]] = None) -> list[int]:
    """N-way peeling split (hb_plan_allocation_n): shares per back-end, in
    back-end order, summing to n_total.  For two back-ends shares ==
    [plan.n_cpu, plan.n_accel] of plan_allocation.  ok = None treats a
    non-positive or non-finite time as a failed back-end (no share)."""
    cnt = len(times)
    t = np.ascontiguousarray(times, dtype=np.float64)
    if ok is None:  # a non-positive / non-finite time marks a failed back-end
        ok = [bool(np.isfinite(x) and x > 0.0) for x in t]
    okv = np.ascontiguousarray([int(b) for b in ok], dtype=np.int32)
    shares = np.zeros(cnt, dtype=np.uint64)
    st = lib.hb_plan_allocation_n(_lib.ptr(t), _lib.ptr(okv), cnt, int(n_total), _lib.ptr(shares))
    if st != _lib.HB_OK:
        raise ValueError(_lib.global_error())
    return [int(s) for s in shares]


def plan_allocation_optimal(cpu_time: Callable[[int], float], accel_time: Callable[[int], float],
                            n_total: int) -> AllocationPlan:
    """Exhaustive min-max oracle, ties toward the smaller accelerator share
    (scheduler.cpp:89-111)."""
    if n_total < 1:
        raise ValueError("plan_allocation_optimal: n_total must be >= 1")
    best_k = 0
    best = max(cpu_time(n_total), accel_time(0))
    for k in range(1, n_total + 1):
        c = max(cpu_time(n_total - k), accel_time(k))
        if c < best:
            best, best_k = c, k
    frac = best_k / n_total
    return AllocationPlan(n_total, n_total - best_k, best_k, frac, frac)


def naive_sum(t_cpu_seq_s: float, t_accel_seq_s: float) -> float:
    if t_cpu_seq_s < 0.0 or t_accel_seq_s < 0.0:
        raise ValueError("naive_sum: times must be >= 0")
    return t_cpu_seq_s + t_accel_seq_s


def format_plan(plan: AllocationPlan) -> str:
    return f"cpu={plan.n_cpu} accel={plan.n_accel}"


def _concat(a: Optional[np.ndarray], b: Optional[np.ndarray]):
    if a is None:
        return b
    if b is None:
        return a
    return np.concatenate([a, b])


def run_hybrid(plan: AllocationPlan, request: BatchRequest, cpu: BatchExecutor,
               accel: BatchExecutor, orchestration_overhead_s: float,
               mode: str = "modeled") -> HybridResult:
    """scheduler.cpp:113-211.  The first n_cpu seeds go to `cpu`, the rest to
    `accel`; "emulated" races both on the real clock (accel on a helper
    thread), "modeled" runs them back to back and composes the wall as
    max(parts) + overhead.  A failing side is re-dispatched to the other and
    the result flagged degraded; both failing re-raises the cpu error."""
    validate_request(request)
    if plan.n_total != len(request.seeds):
        raise ValueError("run_hybrid: plan size does not match request")
    if orchestration_overhead_s < 0.0:
        raise ValueError("run_hybrid: overhead must be >= 0")
    cpu_req = BatchRequest(request.kind, request.seeds[: plan.n_cpu], request.steps)
    acc_req = BatchRequest(request.kind, request.seeds[plan.n_cpu:], request.steps)
    res = {"cpu": None, "accel": None}
    err = {"cpu": None, "accel": None}

    def run_part(side, ex, req):
        try:
            res[side] = ex.run(req)
        except Exception as e:  # noqa: BLE001 - mirrors catch (...)
            err[side] = e

    t0 = time.perf_counter()
    if mode == "emulated":
        th = None
        if plan.n_accel > 0:
            th = threading.Thread(target=run_part, args=("accel", accel, acc_req))
            th.start()
        if plan.n_cpu > 0:
            run_part("cpu", cpu, cpu_req)
        if th is not None:
            th.join()
    else:
        if plan.n_cpu > 0:
            run_part("cpu", cpu, cpu_req)
        if plan.n_accel > 0:
            run_part("accel", accel, acc_req)

    degraded = False
    if err["cpu"] is not None and err["accel"] is not None:
        raise err["cpu"]
    if err["cpu"] is not None:
        degraded = True
        redo = accel.run(cpu_req)
        if res["accel"] is None:
            res["accel"] = redo
        else:
            res["accel"].results = _concat(redo.results, res["accel"].results)
    if err["accel"] is not None:
        degraded = True
        redo = cpu.run(acc_req)
        if res["cpu"] is None:
            res["cpu"] = redo
        else:
            res["cpu"].results = _concat(res["cpu"].results, redo.results)

    out = HybridResult(plan=plan, overhead_s=orchestration_overhead_s, degraded=degraded)
    out.t_cpu_part_s = res["cpu"].wall_time_s if (res["cpu"] and err["cpu"] is None) else 0.0
    out.t_accel_part_s = res["accel"].wall_time_s if (res["accel"] and err["accel"] is None) else 0.0
    if mode == "emulated":
        time.sleep(orchestration_overhead_s)
        out.wall_combined_s = time.perf_counter() - t0
    else:
        out.wall_combined_s = max(out.t_cpu_part_s, out.t_accel_part_s) + orchestration_overhead_s
    out.merged = _concat(res["cpu"].results if res["cpu"] else None,
                         res["accel"].results if res["accel"] else None)
    out.cpu_result = res["cpu"]
    out.accel_result = res["accel"]
    return out


@dataclass
class ShardedResult:
    merged: np.ndarray
    walls: list            # per back-end wall of its (last) part
    wall_s: float          # combined wall clock
    degraded: bool = False
    ok: list = field(default_factory=list)  # per back-end: finished its work

    def __iter__(self):  # (merged, walls, wall) unpacking
        return iter((self.merged, self.walls, self.wall_s))


def run_sharded(shares: Sequence[int], request: BatchRequest,
                executors: Sequence[BatchExecutor]) -> ShardedResult:
    """N-way analogue of run_hybrid (Emulated mode): contiguous slices in
    back-end order, one host thread per back-end, merged in seed order.  A
    back-end that throws anything but BatchFailure is dead for the rest of
    the call; its slice is re-planned over the survivors (plan_allocation_n
    with ok = False for the dead, survivors weighted by their shares) and the
    result is flagged degraded — the N-way form of the reference's
    re-dispatch (scheduler.cpp:162-183).  A BatchFailure is the batch's own
    result (re-running it elsewhere reproduces it) and propagates, as does
    the first error when every back-end has failed."""
    from .executor import BatchFailure
    validate_request(request)
    cnt = len(executors)
    if sum(shares) != len(request.seeds) or len(shares) != cnt:
        raise ValueError("run_sharded: shares do not match the request / executors")
    bounds = np.concatenate([[0], np.cumsum(shares)]).astype(np.int64)
    weights = [1.0 / s if s > 0 else 1.0 for s in shares]
    alive = [True] * cnt
    work = [[(int(bounds[d]), int(bounds[d + 1]))] if shares[d] > 0 else [] for d in range(cnt)]
    parts: dict = {}
    walls = [0.0] * cnt
    first_err = None
    t0 = time.perf_counter()
    while any(work):
        errs: list = [None] * cnt

        def go(d, slices):
            while slices:  # completed slices leave the list; the rest is orphaned on failure
                b, e = slices[0]
                try:
                    r = executors[d].run(BatchRequest(request.kind, request.seeds[b:e], request.steps))
                except Exception as ex:  # noqa: BLE001 - mirrors catch (...)
                    errs[d] = ex
                    return
                parts[b] = r.results
                walls[d] = r.wall_time_s
                slices.pop(0)

        ths = [threading.Thread(target=go, args=(d, work[d])) for d in range(cnt) if work[d]]
        busy = [d for d in range(cnt) if work[d]]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        orphans = []
        for d in busy:
            if errs[d] is None:
                work[d] = []
                continue
            if isinstance(errs[d], BatchFailure):
                raise errs[d]
            first_err = first_err or errs[d]
            alive[d] = False
            orphans.extend(work[d])
            work[d] = []
        if not orphans:
            break
        if not any(alive):
            raise first_err
        for b, e in orphans:
            sub = plan_allocation_n(weights, e - b, alive)
            for d in range(cnt):
                if sub[d]:
                    work[d].append((b, b + sub[d]))
                b += sub[d]
    wall = time.perf_counter() - t0
    merged = np.concatenate([parts[b] for b in sorted(parts)])
    return ShardedResult(merged, walls, wall, not all(alive), list(alive))
