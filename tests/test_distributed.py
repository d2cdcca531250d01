"""World-size-2 gloo tests (CPU) of the multi-process path: per-rank
contiguous shards from the N-way splitter, the fitness all-gather, and the
sharded generation loop — identical to the single-process run_ea."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2502_11129_b200 as hb
from paper_2502_11129_b200 import distributed as hbd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, pop, gens, steps, times, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import OracleExecutor
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = hbd.run_ea_sharded(kind, pop, gens, steps, OracleExecutor(1), dist, seed=3, times=times)
        b = hbd.shard_bounds(1000, world, times)
        q.put((rank, r.population.genomes.tolist(), r.population.fitnesses.tolist(), b.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("times", [None, [1.0, 3.0]])
def test_sharded_ea_world2_equals_single_process(times):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    kind, pop, gens, steps = 1, 64, 3, 40
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, pop, gens, steps, times, q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import OracleExecutor
    ref = hb.run_ea(kind, pop, gens, steps, OracleExecutor(2), seed=3)
    for rank, g, f, b in out:
        assert g == ref.population.genomes.tolist()
        assert np.array_equal(np.array(f), ref.population.fitnesses)
        assert b[0] == 0 and b[-1] == 1000
    expect = hbd.shard_bounds(1000, 2, times).tolist()
    assert all(o[3] == expect for o in out)
    if times is not None:
        assert expect == [0, 750, 1000]  # throughput-proportional (1/t)


def test_shard_bounds_cover_contiguously():
    for world in (1, 2, 3, 8):
        for n in (1, 7, 1000, 65536):
            b = hbd.shard_bounds(n, world)
            assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
            assert np.max(np.diff(b)) - np.min(np.diff(b)) <= world


def _calib_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import OracleExecutor
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        times = hbd.calibrate_ranks(1, 30, 64, OracleExecutor(1), dist, repeats=2)
        q.put((rank, times, [int(x) for x in hb.plan_allocation_n(times, 1000)]))
    finally:
        dist.destroy_process_group()


def test_calibrate_ranks_world2_same_times_and_shares():
    """Every rank times the probe on its own back-end; all ranks end with the
    same time vector and hence the same splitter shares (sum = batch)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_calib_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, t0, s0), (_, t1, s1) = out
    assert t0 == t1 and len(t0) == 2 and all(t > 0 for t in t0)
    assert s0 == s1 and sum(s0) == 1000


def _calib8_worker(rank, world, port, base, fail_rank, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import FailingExecutor, NoisyStubExecutor
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = FailingExecutor() if rank == fail_rank else NoisyStubExecutor(base[rank], 0.03, seed=17 + rank)
        times = hbd.calibrate_ranks(1, 30, 64, ex, dist, repeats=5)
        q.put((rank, times, [int(x) for x in hb.plan_allocation_n(times, 65536)],
               hbd.shard_bounds(65536, world, times).tolist()))
    finally:
        dist.destroy_process_group()


def _run_world8(base, fail_rank=-1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_calib8_worker, args=(r, 8, port, base, fail_rank, q)) for r in range(8)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(8))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o[1] == out[0][1] and o[2] == out[0][2] and o[3] == out[0][3] for o in out)
    return out[0][1], out[0][2]


def test_calibrate_ranks_world8_equal_devices_get_equal_shares():
    """8 identical devices whose probe times jitter by +-3 %: the medians
    agree within the measured spread, so the times snap to equal and the
    65 536 variants split 8192 each (no noise-driven imbalance)."""
    times, shares = _run_world8([1e-3] * 8)
    assert len(set(times)) == 1
    assert shares == [8192] * 8


def test_calibrate_ranks_world8_unequal_devices_proportional():
    """Devices 1x / 2x / 4x slower (with the same jitter): no snapping; each
    rank's share follows its measured throughput 1 / t."""
    base = [1e-3, 1e-3, 2e-3, 2e-3, 1e-3, 1e-3, 4e-3, 4e-3]
    times, shares = _run_world8(base)
    assert sum(shares) == 65536
    expect = np.array([1.0 / b for b in base])
    expect = 65536 * expect / expect.sum()
    assert np.all(np.abs(np.array(shares) - expect) / expect < 0.05)
    assert shares[0] > 1.8 * shares[2] and shares[2] > 1.8 * shares[6]


def test_calibrate_ranks_world8_failing_rank_is_dead():
    """A rank whose back-end throws during calibration gets time 0 and no
    share (scheduler.cpp:40-49); the other 7 split the batch evenly."""
    times, shares = _run_world8([1e-3] * 8, fail_rank=5)
    assert times[5] == 0.0 and shares[5] == 0
    assert sum(shares) == 65536
    live = [s for i, s in enumerate(shares) if i != 5]
    assert max(live) - min(live) <= 1
