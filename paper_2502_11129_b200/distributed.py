"""One process per GPU: the generation loop sharded over ranks.

Variants are independent, so each rank simulates a contiguous slice of every
batch (shares from the N-way splitter, ``plan_allocation_n``) and the only
cross-rank traffic is the per-generation fitness all-gather (8 B / variant)
— over NCCL on NVLink for GPU ranks, gloo in the CPU tests.  Every rank
then performs the identical, deterministic selection (stable descending
sort) and variation, so all ranks hold the same population without any
further exchange.  Genomes and fitness match ``run_ea`` (ea.cpp:33-105)
bit for bit for any world size.
"""
from __future__ import annotations

import time

import numpy as np

from .ea import (K_CHILD_KEY, K_INIT_KEY, EaResult, PhaseProfile, Population, rng_at,
                 stable_order_desc)
from .executor import BatchExecutor, BatchRequest, ModelKind
from .scheduler import plan_allocation_n


def shard_bounds(n: int, world: int, times=None) -> np.ndarray:
    """Contiguous per-rank slice bounds [b_0 = 0, ..., b_world = n] from the
    N-way splitter over calibrated per-rank times (None = equal ranks; a
    time of 0 = a rank that failed calibration, which gets no share)."""
    shares = plan_allocation_n(list(times) if times is not None else [1.0] * world, n)
    return np.concatenate([[0], np.cumsum(shares)]).astype(np.int64)


def calibrate_ranks(kind: ModelKind, steps: int, probe_n: int, executor: BatchExecutor, dist,
                    repeats: int = 5, snap_tol: float = 0.01):
    """The paper's calibration step (scheduler.cpp:30-56) across the ranks of
    the default group: every rank times the same probe (seeds 0..probe_n-1)
    on its own device at once and the per-rank (time, spread, ok) triples are
    all-gathered, so every rank holds the same times — the input of the N-way
    splitter (plan_allocation_n / shard_bounds), which gives each rank a share
    in proportion to its measured throughput.

    A GPU rank times the probe with CUDA events on its context's stream
    (hb_calibrate: relaunched until a sample spans >= 5 ms, median of
    `repeats` samples, relative spread); any other back-end reports the
    median of `repeats` drop-in wall times.  A rank whose back-end throws is
    dead to the splitter (time 0, no share), as a throwing back-end is to
    calibrate (scheduler.cpp:40-49) — the job goes on without it.  Times that
    agree within the largest measured spread (at least snap_tol) snap to
    equal (snap_equal_times): identical GPUs get identical shares instead of
    a split that follows measurement noise."""
    import torch

    from .executor import GpuExecutor
    from .scheduler import median_and_spread, snap_equal_times
    if probe_n < 1:
        raise ValueError("calibrate: probe_n must be >= 1")
    try:
        if isinstance(executor, GpuExecutor):
            t, sp = executor.ctx.calibrate(kind, steps, probe_n, repeats)
        else:
            req = BatchRequest(kind, np.arange(probe_n, dtype=np.uint64), steps)
            t, sp = median_and_spread([executor.run(req).wall_time_s for _ in range(max(1, repeats))])
        ok = 1.0
    except Exception:  # noqa: BLE001 - a failing rank is dead, not fatal
        t, sp, ok = 0.0, 0.0, 0.0
    world = dist.get_world_size()
    mine = torch.tensor([t, sp, ok], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        mine = mine.cuda()
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    rows = [[float(x) for x in p.cpu()] for p in parts]
    oks = [r[2] > 0.5 for r in rows]
    if not any(oks):
        raise RuntimeError("calibrate: all ranks failed")
    times = snap_equal_times([r[0] for r in rows], [r[1] for r in rows], oks, snap_tol)
    return [t if o else 0.0 for t, o in zip(times, oks)]


def evaluate_sharded(kind: ModelKind, genomes: np.ndarray, steps: int, executor: BatchExecutor,
                     dist, device=None, times=None) -> np.ndarray:
    """Fitness of every genome; this rank simulates only its slice."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    b = shard_bounds(len(genomes), world, times)
    mine = genomes[b[rank]:b[rank + 1]]
    if len(mine):
        fit = np.ascontiguousarray(executor.run(BatchRequest(kind, mine, steps)).results["fitness"])
    else:
        fit = np.zeros(0)
    width = int(np.max(np.diff(b)))
    buf = torch.zeros(width, dtype=torch.float64)
    buf[: len(fit)] = torch.from_numpy(fit)
    if device is not None:
        buf = buf.to(device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return np.concatenate([parts[r][: b[r + 1] - b[r]].cpu().numpy() for r in range(world)])


def run_ea_sharded(kind: ModelKind, population_size: int, generations: int, steps: int,
                   executor: BatchExecutor, dist, seed: int = 0, device=None,
                   times=None) -> EaResult:
    """run_ea with each generation's evaluation sharded over the ranks of the
    default process group (torch.distributed)."""
    if population_size < 2 or population_size % 2 != 0:
        raise ValueError("run_ea: population_size must be even and >= 2")
    if generations < 1:
        raise ValueError("run_ea: generations must be >= 1")
    clock = time.perf_counter
    prof = PhaseProfile()
    t_start = clock()
    pop = Population()
    pop.genomes = rng_at(np.uint64(seed) ^ np.uint64(K_INIT_KEY),
                         np.arange(population_size, dtype=np.uint64))
    t0 = clock()
    pop.fitnesses = evaluate_sharded(kind, pop.genomes, steps, executor, dist, device, times)
    prof.evaluation_s += clock() - t0
    mu = population_size // 2
    for g in range(1, generations + 1):
        t0 = clock()
        order = stable_order_desc(pop.fitnesses)[:mu]
        parents, parent_fit = pop.genomes[order], pop.fitnesses[order]
        prof.selection_s += clock() - t0
        t0 = clock()
        ctr = (np.uint64(g) << np.uint64(32)) + np.arange(mu, dtype=np.uint64)
        offspring = rng_at(parents ^ np.uint64(K_CHILD_KEY), ctr)
        prof.variation_s += clock() - t0
        t0 = clock()
        off_fit = evaluate_sharded(kind, offspring, steps, executor, dist, device, times)
        prof.evaluation_s += clock() - t0
        pop.genomes = np.concatenate([parents, offspring])
        pop.fitnesses = np.concatenate([parent_fit, off_fit])
        pop.generation = g
    prof.total_s = clock() - t_start
    acc = prof.selection_s + prof.variation_s + prof.evaluation_s
    prof.bookkeeping_s = max(prof.total_s - acc, 0.0)
    return EaResult(pop, prof, float(np.max(pop.fitnesses)))


def run_ea_sharded_device(kind: ModelKind, population_size: int, generations: int, steps: int,
                          executor, dist, seed: int = 0, times=None) -> EaResult:
    """The generation loop device-resident on every rank (one process per GPU).

    Genomes and fitness live in each rank's HBM.  Per generation: this rank
    evaluates its contiguous slice of the offspring from device memory
    (hb_eval_device: device-side Box init / host initialiser, one stepping
    launch); the fitness slices — plus each slice's blow-up count — are
    all-gathered (NCCL over NVLink: 8 B / variant); every rank then runs the
    identical device selection + variation (hb_ea_select_vary: stable radix
    sort, parent gather, offspring hashing), so the populations stay equal
    without any further exchange and nothing crosses to the host until the
    end.  A blow-up anywhere aborts the loop on every rank, as batch_failure
    aborts run_ea (ea.cpp:25).  Bit-identical to run_ea for any world size.
    With a gloo group (tests: several ranks on one GPU) the all-gather goes
    through host tensors.  hb_* calls run on the context's stream and torch
    work on torch's current stream; the two are joined by host syncs at the
    hand-overs (three per generation, a few µs each)."""
    import ctypes as C

    import torch

    from . import _lib
    from ._lib import lib

    if population_size < 2 or population_size % 2 != 0:
        raise ValueError("run_ea: population_size must be even and >= 2")
    if generations < 1:
        raise ValueError("run_ea: generations must be >= 1")
    ctx = executor.ctx
    dev = torch.device("cuda", ctx.device)
    rank, world = dist.get_rank(), dist.get_world_size()
    host_coll = dist.get_backend() == "gloo"
    clock = time.perf_counter
    prof = PhaseProfile()
    t_start = clock()
    pop_n, mu = population_size, population_size // 2

    def evaluate(src, dst, n):
        b = shard_bounds(n, world, times)
        lo, hi = int(b[rank]), int(b[rank + 1])
        width = int(np.max(np.diff(b)))
        part = bufs[width]  # [fitness..., failures], reused across generations
        failed = C.c_uint64(0)
        if hi > lo:
            # the context's stream; returns after synchronising it (blow-up count read)
            st = lib.hb_eval_device(ctx.handle, int(kind), src.data_ptr() + 8 * lo, hi - lo, int(steps),
                                    part.data_ptr(), C.byref(failed))
            if st not in (_lib.HB_OK, _lib.HB_BLOWUP_PARTIAL):
                raise RuntimeError(f"hb_eval_device failed [{st}]: {ctx.error()}")
        part[width] = float(failed.value)
        if host_coll:
            src_part = part.cpu()
            parts = [torch.empty_like(src_part) for _ in range(world)]
            dist.all_gather(parts, src_part)
        else:
            flat = flats[width]
            dist.all_gather_into_tensor(flat, part)
            parts = list(flat.view(world, width + 1))
        n_failed = int(torch.stack([p[width] for p in parts]).sum().item())  # one D2H per generation
        if n_failed:
            raise RuntimeError(f"run_ea: numerical blow-up during evaluation ({n_failed} variants)")
        dst[:n].copy_(torch.cat([parts[r][: int(b[r + 1] - b[r])] for r in range(world)]).to(dev))
        # hb_* calls run on the context's stream: finish torch's work first
        torch.cuda.current_stream(dev).synchronize()

    widths = {int(np.max(np.diff(shard_bounds(n, world, times)))) for n in (pop_n, mu)}
    bufs = {w: torch.zeros(w + 1, dtype=torch.float64, device=dev) for w in widths}
    flats = {w: torch.empty(world * (w + 1), dtype=torch.float64, device=dev) for w in widths}
    gen = [torch.empty(pop_n, dtype=torch.int64, device=dev) for _ in range(2)]
    fit = [torch.empty(pop_n, dtype=torch.float64, device=dev) for _ in range(2)]
    torch.cuda.current_stream(dev).synchronize()  # buffers allocated before the context uses them
    ctx.check(lib.hb_ea_init_genomes(ctx.handle, int(seed), pop_n, gen[0].data_ptr()), "init genomes")
    t0 = clock()
    evaluate(gen[0], fit[0], pop_n)
    prof.evaluation_s += clock() - t0
    cur = 0
    for g in range(1, generations + 1):
        nxt = cur ^ 1
        t0 = clock()
        ctx.check(lib.hb_ea_select_vary(ctx.handle, gen[cur].data_ptr(), fit[cur].data_ptr(), pop_n, g,
                                        gen[nxt].data_ptr(), fit[nxt].data_ptr()), "select/vary")
        prof.selection_s += clock() - t0
        t0 = clock()
        evaluate(gen[nxt][mu:], fit[nxt][mu:], mu)
        prof.evaluation_s += clock() - t0
        cur = nxt
    ctx.synchronize()
    genomes = gen[cur].cpu().numpy().view(np.uint64).copy()
    fitness = fit[cur].cpu().numpy().copy()
    prof.total_s = clock() - t_start
    acc = prof.selection_s + prof.variation_s + prof.evaluation_s
    prof.bookkeeping_s = max(prof.total_s - acc, 0.0)
    pop = Population(genomes, fitness, generations)
    return EaResult(pop, prof, float(np.max(fitness)))
