"""(mu + lambda) generation loop — mirror of /root/reference/proj/src/ea.cpp:33-145.

Genomes are variant seeds.  Each generation: evaluate through any
BatchExecutor (the GPU executors here), select the top half by a stable
descending sort of fitness (std::stable_sort with `>`, ea.cpp:60-66), derive
offspring ``rng::at(parent ^ kChildKey, (g << 32) + i)`` (ea.cpp:75-79) and
evaluate them.  The trajectory is a pure function of the arguments, so the
genomes and fitness of every generation are bit-identical to the reference's
run_ea over its cpu_executor.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import lib
from .executor import BatchExecutor, BatchRequest, GpuExecutor, ModelKind, MultiGpuExecutor

K_INIT_KEY = 0x8F5D4C3B2A190807
K_CHILD_KEY = 0x243F6A8885A308D3
_INC = np.uint64(0x9E3779B97F4A7C15)


def _mix64(x: np.ndarray) -> np.ndarray:
    """rng::mix64 (rng.hpp:15-22), vectorised over uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def rng_at(key, counter) -> np.ndarray:
    """rng::at (rng.hpp:25-27), vectorised."""
    key = np.asarray(key, dtype=np.uint64)
    counter = np.asarray(counter, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix64(_mix64(key + _INC) ^ (counter * np.uint64(0xD1B54A32D192ED03) + np.uint64(1)))


def stable_order_desc(fitness: np.ndarray) -> np.ndarray:
    """Index order of std::stable_sort(order, fitness[a] > fitness[b])
    (ea.cpp:60-66) for non-NaN fitness: ties keep input order."""
    return np.argsort(-np.asarray(fitness, dtype=np.float64), kind="stable")


@dataclass
class Population:
    genomes: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))
    fitnesses: np.ndarray = field(default_factory=lambda: np.zeros(0))
    generation: int = 0


@dataclass
class PhaseProfile:
    selection_s: float = 0.0
    variation_s: float = 0.0
    evaluation_s: float = 0.0
    bookkeeping_s: float = 0.0
    total_s: float = 0.0
    # native loop only: wall time not covered by device work (host launch,
    # sync and bookkeeping cost); not part of ea.cpp's profile
    host_overhead_s: float = 0.0

    def evaluation_fraction(self) -> float:
        return self.evaluation_s / self.total_s if self.total_s > 0.0 else 0.0


@dataclass
class EaResult:
    population: Population
    profile: PhaseProfile
    best_fitness: float
    history: list = field(default_factory=list)  # per generation: (genomes, fitnesses)


def _evaluate(kind, genomes, steps, executor: BatchExecutor) -> np.ndarray:
    res = executor.run(BatchRequest(kind, genomes, steps))
    return np.ascontiguousarray(res.results["fitness"])


def run_ea(kind: ModelKind, population_size: int, generations: int, steps: int,
           executor: BatchExecutor, seed: int = 0, keep_history: bool = False,
           native: bool = True) -> EaResult:
    """ea.cpp:33-105.  With a GPU executor (and native=True) the whole loop runs
    natively (hb_run_ea: device-side selection / variation, offspring sharded
    over the executor's devices); any other BatchExecutor goes through the
    same loop in Python."""
    if native and isinstance(executor, (GpuExecutor, MultiGpuExecutor)):
        return run_ea_native(kind, population_size, generations, steps, executor, seed, keep_history)
    if population_size < 2 or population_size % 2 != 0:
        raise ValueError("run_ea: population_size must be even and >= 2")
    if generations < 1:
        raise ValueError("run_ea: generations must be >= 1")
    prof = PhaseProfile()
    clock = time.perf_counter
    t_start = clock()
    history = []

    t0 = clock()
    pop = Population()
    pop.genomes = rng_at(np.uint64(seed) ^ np.uint64(K_INIT_KEY),
                         np.arange(population_size, dtype=np.uint64))
    prof.bookkeeping_s += clock() - t0
    t0 = clock()
    pop.fitnesses = _evaluate(kind, pop.genomes, steps, executor)
    prof.evaluation_s += clock() - t0
    if keep_history:
        history.append((pop.genomes.copy(), pop.fitnesses.copy()))

    mu = population_size // 2
    for g in range(1, generations + 1):
        t0 = clock()
        order = stable_order_desc(pop.fitnesses)[:mu]
        parents = pop.genomes[order]
        parent_fitness = pop.fitnesses[order]
        prof.selection_s += clock() - t0

        t0 = clock()
        ctr = (np.uint64(g) << np.uint64(32)) + np.arange(mu, dtype=np.uint64)
        offspring = rng_at(parents ^ np.uint64(K_CHILD_KEY), ctr)
        prof.variation_s += clock() - t0

        t0 = clock()
        off_fit = _evaluate(kind, offspring, steps, executor)
        prof.evaluation_s += clock() - t0

        t0 = clock()
        pop.genomes = np.concatenate([parents, offspring])
        pop.fitnesses = np.concatenate([parent_fitness, off_fit])
        pop.generation = g
        prof.bookkeeping_s += clock() - t0
        if keep_history:
            history.append((pop.genomes.copy(), pop.fitnesses.copy()))

    prof.total_s = clock() - t_start
    accounted = prof.selection_s + prof.variation_s + prof.evaluation_s + prof.bookkeeping_s
    if prof.total_s > accounted:
        prof.bookkeeping_s += prof.total_s - accounted
    return EaResult(pop, prof, float(np.max(pop.fitnesses)), history)


def run_ea_native(kind: ModelKind, population_size: int, generations: int, steps: int,
                  executor, seed: int = 0, keep_history: bool = False,
                  device_times=None) -> EaResult:
    """hb_run_ea over the executor's device contexts."""
    if population_size < 2 or population_size % 2 != 0:
        raise ValueError("run_ea: population_size must be even and >= 2")
    if generations < 1:
        raise ValueError("run_ea: generations must be >= 1")
    ctxs = [executor.ctx] if isinstance(executor, GpuExecutor) else list(executor.ctxs)
    cnt = len(ctxs)
    handles = (C.c_void_p * cnt)(*[c.handle for c in ctxs])
    times = None
    if device_times is None and isinstance(executor, MultiGpuExecutor):
        # the executor's calibration: measured per-device probe times, else
        # its fixed shares read as throughputs (time ~ 1 / share; a device
        # with no share gets an infinite time, hence no offspring)
        if executor.device_times is not None:
            device_times = executor.device_times
        elif executor.shares is not None:
            device_times = [1.0 / s if s > 0 else np.inf for s in executor.shares]
    if device_times is not None:
        times = np.ascontiguousarray(device_times, dtype=np.float64)
        if len(times) != cnt:
            raise ValueError("run_ea: one device time per context required")
    # page-locked (recycled) outputs: the final population is DMA'd straight in
    gen = _lib.pinned.empty(population_size, np.uint64)
    fit = _lib.pinned.empty(population_size, np.float64)
    best = C.c_double(0)
    prof = _lib.PhaseProfile()
    hg = hf = None
    if keep_history:
        hg = np.empty((generations + 1, population_size), dtype=np.uint64)
        hf = np.empty((generations + 1, population_size))
    st = lib.hb_run_ea(C.cast(handles, C.c_void_p), cnt, None if times is None else _lib.ptr(times),
                       int(kind), population_size, int(generations), int(steps), int(seed),
                       _lib.ptr(gen), _lib.ptr(fit), C.byref(best), C.byref(prof),
                       None if hg is None else _lib.ptr(hg), None if hf is None else _lib.ptr(hf))
    if st == _lib.HB_INVALID_ARG:
        raise ValueError(ctxs[0].error())
    if st == _lib.HB_BLOWUP_PARTIAL:
        raise RuntimeError(ctxs[0].error())
    if st != _lib.HB_OK:
        raise RuntimeError(f"hb_run_ea failed [{st}]: {ctxs[0].error()}")
    profile = PhaseProfile(prof.selection_s, prof.variation_s, prof.evaluation_s,
                           prof.bookkeeping_s, prof.total_s, prof.host_overhead_s)
    history = [] if hg is None else [(hg[g], hf[g]) for g in range(generations + 1)]
    return EaResult(Population(gen, fit, generations), profile, float(best.value), history)


def report_profile(profile: PhaseProfile) -> str:
    """ea.cpp:107-145: phase table sorted by seconds (stable), then
    profile.<key>=<%.9g> lines."""
    rows = [("selection", profile.selection_s), ("variation", profile.variation_s),
            ("evaluation", profile.evaluation_s), ("bookkeeping", profile.bookkeeping_s)]
    rows = sorted(rows, key=lambda r: -r[1])  # Python sort is stable
    total = profile.total_s
    out = ["%-12s %12s %9s\n" % ("phase", "seconds", "fraction")]
    for name, secs in rows:
        out.append("%-12s %12.6f %9.3f\n" % (name, secs, secs / total if total > 0.0 else 0.0))
    out.append("%-12s %12.6f %9.3f\n" % ("total", total, 1.0 if total > 0.0 else 0.0))
    for key, v in (("selection_s", profile.selection_s), ("variation_s", profile.variation_s),
                   ("evaluation_s", profile.evaluation_s), ("bookkeeping_s", profile.bookkeeping_s),
                   ("total_s", profile.total_s),
                   ("evaluation_fraction", profile.evaluation_fraction())):
        out.append("profile.%s=%s\n" % (key, _g9(v)))
    return "".join(out)


def _g9(v: float) -> str:
    return "%.9g" % v
