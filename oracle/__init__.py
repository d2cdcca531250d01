"""TEST INFRASTRUCTURE ONLY — the parity oracle.

ctypes bindings for
  * ``_build/libhboracle.so`` — the plain-C restatement (hb_oracle.c), and
  * ``_ref/libhetbench_ref.so`` — the unmodified reference sources compiled
    in place (ref_shim.cpp), present when built in the dev container and
    shipped prebuilt to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference arm may import this package.  The product package
(``paper_2502_11129_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhetbench_ref.so")

BOX, BOX_AND_BALL, ARM_WITH_ROPE, HUMANOID, CPG_HINGE = 0, 1, 2, 3, 4
MODEL_NAMES = ("box", "box_and_ball", "arm_with_rope", "humanoid", "cpg_hinge")
BODIES = (1, 2, 12, 32, 9)
CONSTRAINTS = (0, 1, 11, 46, 12)
DT = 0.002

RESULT_DTYPE = np.dtype([("seed", "<u8"), ("fitness", "<f8"), ("checksum", "<u8"),
                         ("steps_executed", "<u8")])


class _Result(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("fitness", C.c_double), ("checksum", C.c_uint64),
                ("steps_executed", C.c_uint64)]


class _Plan(C.Structure):
    _fields_ = [("n_total", C.c_uint64), ("n_cpu", C.c_uint64), ("n_accel", C.c_uint64),
                ("accel_fraction", C.c_double), ("requested_accel_fraction", C.c_double)]


def build(with_ref: bool | None = None) -> None:
    """Compile the oracle (and the reference library when /root/reference exists)."""
    target = "all" if with_ref is None else ("ref" if with_ref else "oracle")
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def _load(path: str):
    if not os.path.exists(path):
        build(with_ref=None)
    return C.CDLL(path)


_orc = None
_ref = None


def lib():
    global _orc
    if _orc is None:
        _orc = _load(ORACLE_SO)
        L = _orc
        u64, dbl, i32, sz = C.c_uint64, C.c_double, C.c_int, C.c_size_t
        p = C.POINTER
        L.hbo_rng_at.restype = u64
        L.hbo_rng_at.argtypes = [u64, u64]
        L.hbo_mix64.restype = u64
        L.hbo_mix64.argtypes = [u64]
        L.hbo_build_model.argtypes = [i32, u64, p(dbl), p(dbl), p(dbl)]
        L.hbo_step.argtypes = [i32, p(dbl), p(dbl), p(dbl), dbl, p(dbl)]
        L.hbo_checksum.restype = u64
        L.hbo_checksum.argtypes = [i32, p(dbl), p(dbl)]
        L.hbo_simulate.argtypes = [i32, u64, u64, p(_Result), p(u64)]
        L.hbo_simulate_batch.argtypes = [i32, p(u64), sz, u64, i32, C.c_void_p, p(u64)]
        L.hbo_plan_allocation.argtypes = [dbl, dbl, i32, i32, u64, p(_Plan)]
        L.hbo_stable_order_desc.argtypes = [p(dbl), sz, p(sz)]
        L.hbo_time_after.restype = dbl
        L.hbo_time_after.argtypes = [u64, dbl]
        L.hbo_blowup_message.argtypes = [u64, u64, dbl, C.c_char_p, sz]
        L.hbo_run_ea.argtypes = [i32, sz, u64, u64, u64, i32, p(u64), p(dbl)]
        L.hbo_cpg_build.argtypes = [u64, p(dbl), p(dbl), p(dbl), p(dbl)]
        L.hbo_cpg_step.argtypes = [p(dbl), p(dbl), p(dbl), p(dbl), dbl, p(dbl)]
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference library itself (None if it was never built here)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            return None
        _ref = C.CDLL(REF_SO)
        L = _ref
        u64, dbl, i32, sz = C.c_uint64, C.c_double, C.c_int, C.c_size_t
        p = C.POINTER
        L.hbref_hardware_concurrency.restype = C.c_uint
        L.hbref_simulate.argtypes = [i32, u64, u64, p(_Result), C.c_char_p, sz]
        L.hbref_build_model.argtypes = [i32, u64, p(dbl), p(dbl), p(dbl), p(u64), p(u64), p(dbl)]
        L.hbref_trajectory.argtypes = [i32, u64, u64, p(dbl), p(dbl), p(dbl)]
        L.hbref_step_state.argtypes = [i32, p(dbl), p(dbl), dbl, u64, C.c_char_p, sz]
        L.hbref_state_checksum.restype = u64
        L.hbref_state_checksum.argtypes = [i32, u64]
        L.hbref_cpu_run.argtypes = [i32, p(u64), sz, u64, C.c_uint, C.c_void_p, p(dbl), p(u64),
                                    p(sz), C.c_char_p, sz]
        L.hbref_plan_allocation.argtypes = [dbl, dbl, i32, i32, u64, p(_Plan)]
        L.hbref_run_ea.argtypes = [i32, sz, u64, u64, u64, C.c_uint, p(u64), p(dbl), p(dbl)]
        L.hbref_detect_knee.argtypes = [p(u64), p(dbl), sz, dbl, p(u64), p(i32)]
        L.hbref_blowup_after.argtypes = [i32, u64, u64, C.c_char_p, sz]
        L.hbref_rng_at.restype = u64
        L.hbref_rng_at.argtypes = [u64, u64]
    return _ref


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# ---------------------------------------------------------------- restatement
def rng_at(key: int, ctr: int) -> int:
    return int(lib().hbo_rng_at(key, ctr))


def build_model(kind: int, seed: int):
    n, m = BODIES[kind], CONSTRAINTS[kind]
    pos = np.zeros((n, 3)); vel = np.zeros((n, 3)); rest = np.zeros(max(m, 1))
    lib().hbo_build_model(kind, seed, _dp(pos), _dp(vel), _dp(rest))
    return pos, vel, rest[:m]


def cpg_build(seed: int):
    """CpgHinge initial state (not in the reference): pos (9,3), vel (9,3),
    rest (12,) with L0 in 8..11, cpg (16,) = x[4], y[4], omega[4], coupling[4]."""
    pos = np.zeros((9, 3)); vel = np.zeros((9, 3)); rest = np.zeros(12); cpg = np.zeros(16)
    lib().hbo_cpg_build(seed, _dp(pos), _dp(vel), _dp(rest), _dp(cpg))
    return pos, vel, rest, cpg


def cpg_step(pos, vel, rest, cpg, dt: float = DT, time: float = 0.0):
    t = C.c_double(time)
    rc = lib().hbo_cpg_step(_dp(pos), _dp(vel), _dp(rest), _dp(cpg), dt, C.byref(t))
    return rc, t.value


def step(kind: int, pos, vel, rest, dt: float = DT, time: float = 0.0):
    """One reference step on (pos, vel) in place.  Returns (rc, time)."""
    t = C.c_double(time)
    r = np.ascontiguousarray(rest if len(rest) else np.zeros(1))
    rc = lib().hbo_step(kind, _dp(pos), _dp(vel), _dp(r), dt, C.byref(t))
    return rc, t.value


def checksum(pos, vel) -> int:
    return int(lib().hbo_checksum(pos.shape[0], _dp(pos), _dp(vel)))


@dataclass
class OracleBatch:
    results: np.ndarray      # RESULT_DTYPE
    fail_step: np.ndarray    # u64, 0 = ok


def simulate(kind: int, seed: int, steps: int):
    r = _Result()
    fs = C.c_uint64(0)
    rc = lib().hbo_simulate(kind, seed, steps, C.byref(r), C.byref(fs))
    if rc < 0:
        raise ValueError("simulate: steps must be >= 1")
    return rc, (r.seed, r.fitness, r.checksum, r.steps_executed), fs.value


def simulate_batch(kind: int, seeds, steps: int, threads: int | None = None) -> OracleBatch:
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.zeros(len(seeds), dtype=RESULT_DTYPE)
    fail = np.zeros(len(seeds), dtype=np.uint64)
    threads = threads or os.cpu_count() or 1
    rc = lib().hbo_simulate_batch(kind, _up(seeds), len(seeds), steps, threads,
                                  out.ctypes.data_as(C.c_void_p), _up(fail))
    if rc < 0:
        raise ValueError("simulate_batch: bad arguments")
    return OracleBatch(out, fail)


def blowup_message(seed: int, fail_step: int, dt: float = DT) -> str:
    buf = C.create_string_buffer(256)
    lib().hbo_blowup_message(seed, fail_step, dt, buf, 256)
    return buf.value.decode()


def plan_allocation(t_cpu, t_accel, n_total, cpu_ok=True, accel_ok=True):
    p = _Plan()
    if lib().hbo_plan_allocation(t_cpu, t_accel, int(cpu_ok), int(accel_ok), n_total, C.byref(p)):
        raise ValueError("plan_allocation: n_total must be >= 1")
    return (p.n_total, p.n_cpu, p.n_accel, p.accel_fraction, p.requested_accel_fraction)


def stable_order_desc(fitness) -> np.ndarray:
    f = np.ascontiguousarray(fitness, dtype=np.float64)
    order = np.zeros(len(f), dtype=np.uintp)
    lib().hbo_stable_order_desc(_dp(f), len(f), order.ctypes.data_as(C.POINTER(C.c_size_t)))
    return order.astype(np.int64)


def run_ea(kind, pop, generations, steps, seed=0, threads=None):
    g = np.zeros(pop, dtype=np.uint64)
    f = np.zeros(pop)
    rc = lib().hbo_run_ea(kind, pop, generations, steps, seed, threads or os.cpu_count() or 1,
                          _up(g), _dp(f))
    if rc < 0:
        raise ValueError("run_ea: bad arguments")
    if rc == 1:
        raise RuntimeError("run_ea: blow-up")
    return g, f


# ------------------------------------------------------------------ reference
def ref_simulate(kind: int, seed: int, steps: int):
    L = ref()
    r = _Result()
    buf = C.create_string_buffer(512)
    rc = L.hbref_simulate(kind, seed, steps, C.byref(r), buf, 512)
    return rc, (r.seed, r.fitness, r.checksum, r.steps_executed), buf.value.decode()


def ref_cpu_run(kind: int, seeds, steps: int, workers: int = 0):
    """Reference cpu_executor(workers, monitor=false).run.  Returns
    (rc, results, wall_s, failed_seeds, message)."""
    L = ref()
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.zeros(len(seeds), dtype=RESULT_DTYPE)
    wall = C.c_double(0)
    failed = np.zeros(len(seeds), dtype=np.uint64)
    nf = C.c_size_t(0)
    buf = C.create_string_buffer(1024)
    rc = L.hbref_cpu_run(kind, _up(seeds), len(seeds), steps, workers,
                         out.ctypes.data_as(C.c_void_p), C.byref(wall), _up(failed),
                         C.byref(nf), buf, 1024)
    return rc, out, wall.value, failed[: nf.value], buf.value.decode()


def ref_plan_allocation(t_cpu, t_accel, n_total, cpu_ok=True, accel_ok=True):
    p = _Plan()
    ref().hbref_plan_allocation(t_cpu, t_accel, int(cpu_ok), int(accel_ok), n_total, C.byref(p))
    return (p.n_total, p.n_cpu, p.n_accel, p.accel_fraction, p.requested_accel_fraction)


def ref_run_ea(kind, pop, generations, steps, seed=0, workers=0):
    g = np.zeros(pop, dtype=np.uint64)
    f = np.zeros(pop)
    best = C.c_double(0)
    rc = ref().hbref_run_ea(kind, pop, generations, steps, seed, workers, _up(g), _dp(f),
                            C.byref(best))
    if rc:
        raise RuntimeError("reference run_ea failed")
    return g, f


def ref_hardware_concurrency() -> int:
    return int(ref().hbref_hardware_concurrency())
