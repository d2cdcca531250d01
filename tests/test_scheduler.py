"""Splitter (scheduler.cpp) against the reference's own scheduler tests
(proj/tests/test_scheduler.cpp) with stub back-ends."""
import numpy as np
import pytest

import paper_2502_11129_b200 as hb
from helpers import FailingExecutor, OracleExecutor, StubExecutor


def profile_from(t_cpu, t_accel):
    return hb.CalibrationProfile(hb.ModelKind.Box, 100, 8, t_cpu, t_accel, t_accel / t_cpu)


def request_of(n, steps=60, kind=0):
    return hb.BatchRequest(kind, np.arange(n, dtype=np.uint64), steps)


def test_calibrate_records_walls():
    cpu, acc = StubExecutor(2.0), StubExecutor(2.0)
    p = hb.calibrate(0, 100, 8, cpu, acc)
    assert (p.steps, p.probe_n, p.t_cpu_s, p.t_accel_s, p.ratio_accel_over_cpu) == (100, 8, 2.0, 2.0, 1.0)
    assert p.cpu_ok and p.accel_ok and cpu.calls == 1 and acc.calls == 1
    assert hb.calibrate(0, 100, 8, cpu, StubExecutor(6.0)).ratio_accel_over_cpu == 3.0


def test_calibrate_routes_around_failure():
    good, bad = StubExecutor(2.0), StubExecutor(0.0, fail=True)
    p = hb.calibrate(0, 100, 4, bad, good)
    assert not p.cpu_ok and p.accel_ok
    plan = hb.plan_allocation(p, 10)
    assert (plan.n_cpu, plan.n_accel, plan.requested_accel_fraction) == (0, 10, 1.0)
    p = hb.calibrate(0, 100, 4, good, bad)
    plan = hb.plan_allocation(p, 10)
    assert (plan.n_cpu, plan.n_accel) == (10, 0)
    with pytest.raises(RuntimeError):
        hb.calibrate(0, 100, 4, bad, StubExecutor(0.0, fail=True))
    with pytest.raises(ValueError):
        hb.calibrate(0, 100, 0, good, good)


def test_reference_splits():
    p = hb.plan_allocation(profile_from(2.0, 2.0), 100)
    assert (p.n_cpu, p.n_accel, p.accel_fraction) == (50, 50, 0.5)
    assert hb.plan_allocation(profile_from(2.0, 6.0), 100).n_accel == 25
    assert hb.plan_allocation(profile_from(1.0, 1e9), 10).n_accel == 0
    p = hb.plan_allocation(profile_from(19.0, 1.0), 10)
    assert (p.n_accel, p.n_cpu) == (9, 1)
    assert hb.plan_allocation(profile_from(1.0, 1e-9), 10).n_cpu == 0


def test_heuristic_tracks_optimal():
    rng = np.random.default_rng(0x5EED)
    for _ in range(100):
        a, b = rng.uniform(0.1, 10.0, 2)
        for n in (10, 100, 1000):
            h = hb.plan_allocation(profile_from(a, b), n)
            o = hb.plan_allocation_optimal(lambda k: a * k, lambda k: b * k, n)
            assert abs(h.n_accel - o.n_accel) <= 1


def test_run_hybrid_one_sided():
    req = request_of(12)
    cpu, acc = StubExecutor(0.25, 0.05), StubExecutor(9.9)
    plan = hb.plan_allocation(profile_from(1.0, 1e9), 12)
    hr = hb.run_hybrid(plan, req, cpu, acc, 0.1, "modeled")
    assert acc.calls == 0 and hr.t_cpu_part_s == 0.25 and hr.t_accel_part_s == 0.0
    assert abs(hr.wall_combined_s - 0.35) < 1e-9 and len(hr.merged) == 12 and not hr.degraded


def test_run_hybrid_modeled_composition():
    req = request_of(20)
    plan = hb.plan_allocation(profile_from(1.0, 1.0), 20)
    hr = hb.run_hybrid(plan, req, StubExecutor(0.30), StubExecutor(0.75), 0.1, "modeled")
    assert abs(hr.wall_combined_s - 0.85) < 1e-9
    assert list(hr.merged["seed"]) == list(range(20))


def test_run_hybrid_emulated_concurrency():
    req = request_of(16, 5)
    plan = hb.plan_allocation(profile_from(1.0, 1.0), 16)
    hr = hb.run_hybrid(plan, req, StubExecutor(0.4, 0.4), StubExecutor(0.7, 0.7), 0.1, "emulated")
    assert 0.8 * 0.97 <= hr.wall_combined_s <= 0.8 * 1.1 + 0.05


def test_run_hybrid_merge_equals_sequential():
    req = hb.BatchRequest(1, np.array([11, 3, 7, 19, 2, 5, 23, 1, 13, 17, 0, 29], dtype=np.uint64), 60)
    plan = hb.plan_allocation(profile_from(1.0, 1.0), 12)
    hr = hb.run_hybrid(plan, req, OracleExecutor(), OracleExecutor(1), 0.0, "modeled")
    assert np.array_equal(hr.merged, OracleExecutor(1).run(req).results)


def test_run_hybrid_redispatch():
    req = request_of(16, 30)
    plan = hb.plan_allocation(profile_from(1.0, 1.0), 16)
    ref = OracleExecutor(1).run(req).results
    hr = hb.run_hybrid(plan, req, OracleExecutor(), StubExecutor(0.0, fail=True), 0.02, "modeled")
    assert hr.degraded and hr.t_accel_part_s == 0.0 and np.array_equal(hr.merged, ref)
    hr = hb.run_hybrid(plan, req, StubExecutor(0.0, fail=True), OracleExecutor(), 0.02, "modeled")
    assert hr.degraded and hr.t_cpu_part_s == 0.0 and np.array_equal(hr.merged, ref)
    with pytest.raises(RuntimeError):
        hb.run_hybrid(plan, req, StubExecutor(0.0, fail=True), StubExecutor(0.0, fail=True), 0.0)


def test_run_hybrid_preconditions():
    plan = hb.plan_allocation(profile_from(1.0, 1.0), 8)
    with pytest.raises(ValueError):
        hb.run_hybrid(plan, request_of(9), StubExecutor(1.0), StubExecutor(1.0), 0.0)
    with pytest.raises(ValueError):
        hb.run_hybrid(plan, request_of(8), StubExecutor(1.0), StubExecutor(1.0), -0.1)


def test_naive_sum_and_format():
    assert hb.naive_sum(2.0, 3.0) == 5.0
    with pytest.raises(ValueError):
        hb.naive_sum(-1.0, 0.0)
    assert hb.format_plan(hb.AllocationPlan(100, 75, 25)) == "cpu=75 accel=25"


def test_run_sharded_nway():
    req = request_of(1000, 20, kind=1)
    exs = [OracleExecutor(1) for _ in range(4)]
    shares = hb.plan_allocation_n([1.0, 2.0, 0.5, 1.0], 1000)
    merged, walls, wall = hb.run_sharded(shares, req, exs)
    assert np.array_equal(merged, OracleExecutor(2).run(req).results)
    assert len(walls) == 4 and wall > 0


def test_run_sharded_degraded_redispatch():
    """A back-end that throws is dead: its slice is re-planned over the
    survivors (plan_allocation_n, ok = False) and the merge is identical to a
    healthy run, flagged degraded (scheduler.cpp:162-183, N-way)."""
    req = request_of(1000, 20, kind=1)
    exs = [OracleExecutor(1), FailingExecutor(), OracleExecutor(1), OracleExecutor(1)]
    shares = hb.plan_allocation_n([1.0, 1.0, 2.0, 1.0], 1000)
    r = hb.run_sharded(shares, req, exs)
    assert r.degraded and r.ok == [True, False, True, True]
    assert np.array_equal(r.merged, OracleExecutor(2).run(req).results)
    healthy = hb.run_sharded(shares, req, [OracleExecutor(1) for _ in range(4)])
    assert not healthy.degraded and np.array_equal(healthy.merged, r.merged)
    with pytest.raises(RuntimeError):
        hb.run_sharded([500, 500], request_of(1000, 20, kind=1), [FailingExecutor(), FailingExecutor()])


def test_calibrate_n_marks_failure_and_snaps():
    from helpers import NoisyStubExecutor
    req_kind, steps = 1, 20
    exs = [NoisyStubExecutor(1e-3, 0.03, seed=s) for s in range(4)] + [FailingExecutor()]
    times, ok = hb.calibrate_n(req_kind, steps, 8, exs)
    assert ok == [True] * 4 + [False] and times[4] == 0.0
    assert len(set(times[:4])) == 1  # snapped to equal
    assert hb.plan_allocation_n(times, 1000, ok) == [250, 250, 250, 250, 0]
    t2, _ = hb.calibrate_n(req_kind, steps, 8, [StubExecutor(1.0), StubExecutor(3.0)])
    assert t2 == [1.0, 3.0]
