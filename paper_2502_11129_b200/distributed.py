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
    N-way splitter over calibrated per-rank times (None = equal ranks)."""
    shares = plan_allocation_n(list(times) if times is not None else [1.0] * world, n)
    return np.concatenate([[0], np.cumsum(shares)]).astype(np.int64)


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
