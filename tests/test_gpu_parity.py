"""GPU parity: the CUDA product path (through the C ABI) against the oracle
and the reference's golden vectors.  Bar: bit-exact — fitness bits, checksum,
seed and steps of every VariantResult; identical failure seeds / messages."""
import numpy as np
import pytest

import oracle as O
import paper_2502_11129_b200 as hb

pytestmark = pytest.mark.gpu


def fbits(x):
    return "%016x" % int(np.float64(x).view(np.uint64))


def test_golden_simulate_grid(gpu, golden):
    by = {}
    for g in golden["simulate"]:
        by.setdefault((g["kind"], g["steps"]), []).append(g)
    for (kind, steps), rows in by.items():
        seeds = np.array([int(r["seed"]) for r in rows], dtype=np.uint64)
        res = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
        for r, g in zip(res, rows):
            assert int(r["seed"]) == int(g["seed"])
            assert fbits(r["fitness"]) == g["fitness_bits"], (kind, steps, g["seed"])
            assert "%016x" % int(r["checksum"]) == g["checksum"], (kind, steps, g["seed"])
            assert int(r["steps_executed"]) == steps


def test_acceptance_c1_recipe(gpu, golden):
    """acceptance.cpp:200-218 with the GPU executor in the accelerator slot."""
    groups = {}
    for g in golden["c1"]:
        groups.setdefault((g["kind"], g["steps"]), []).append(g)
    total = 0
    for (kind, steps), rows in groups.items():
        seeds = np.array([int(r["seed"]) for r in rows], dtype=np.uint64)
        res = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
        assert [("%016x" % int(c)) for c in res["checksum"]] == [r["checksum"] for r in rows]
        assert [fbits(f) for f in res["fitness"]] == [r["fitness_bits"] for r in rows]
        total += len(rows)
    assert total == 200


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_random_batches_vs_oracle(gpu, kind):
    rng = np.random.default_rng(100 + kind)
    seeds = rng.integers(0, 2**64 - 1, size=(4096, 2048, 512, 256)[kind], dtype=np.uint64,
                         endpoint=True)
    for steps in (1, 37, 300):
        got = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
        want = O.simulate_batch(kind, seeds, steps)
        assert np.all(want.fail_step == 0)
        assert np.array_equal(got, want.results), (kind, steps)


def test_long_horizon_vs_oracle(gpu):
    # step-count sweep endpoints (config 4 goes to 20 000 steps)
    for kind, n, steps in ((0, 256, 20000), (1, 128, 20000), (2, 32, 5000), (3, 16, 5000)):
        seeds = np.arange(n, dtype=np.uint64) * np.uint64(7919)
        got = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
        want = O.simulate_batch(kind, seeds, steps)
        assert np.array_equal(got, want.results), (kind, steps)


def test_trajectories_vs_golden(gpu, golden):
    """Full final state (positions, velocities) after 1/7/64/500 steps."""
    for g in golden["trajectory"]:
        kind = g["kind"]
        soa = hb.build_states(kind, [int(g["seed"])])
        n, m = O.BODIES[kind], O.CONSTRAINTS[kind]
        pos = soa[: 3 * n, 0].reshape(1, n, 3)
        vel = soa[3 * n: 6 * n, 0].reshape(1, n, 3)
        rest = soa[6 * n:, 0].reshape(1, m)
        out, fail, fp, fv = gpu.run_states(kind, pos, vel, rest, steps=g["steps"])
        assert fail[0] == 0
        assert [fbits(x) for x in fp.ravel()] == g["pos_bits"]
        assert [fbits(x) for x in fv.ravel()] == g["vel_bits"]


def test_known_answers(gpu, golden):
    ka = golden["known_answers"]
    # rest on the ground (test_simkernel.cpp:106-115)
    _, fail, p, v = gpu.run_states(0, [[[0.3, -0.2, 0.0]]], [[[0.0, 0.0, 0.0]]], np.zeros((1, 0)))
    assert fail[0] == 0
    assert [fbits(x) for x in p.ravel()] == ka["rest_on_ground"]["pos_bits"]
    assert v[0, 0, 2] == 0.0
    # damped free-fall kick (:117-126)
    _, fail, p, v = gpu.run_states(0, [[[0.0, 0.0, 5.0]]], [[[0.0, 0.0, 0.0]]], np.zeros((1, 0)))
    expected = -9.81 * 0.002 * (1.0 - 0.8 * 0.002)
    assert abs(v[0, 0, 2] - expected) < 1e-12
    assert [fbits(x) for x in v.ravel()] == ka["free_fall"]["vel_bits"]
    assert [fbits(x) for x in p.ravel()] == ka["free_fall"]["pos_bits"]
    # non-positive dt is rejected (:123)
    with pytest.raises(ValueError, match="dt"):
        gpu.run_states(0, [[[0.0, 0.0, 5.0]]], [[[0.0, 0.0, 0.0]]], np.zeros((1, 0)), dt=0.0)


def test_blowup_surfaces_as_batch_failure(gpu, golden):
    """v.z = 1e9 blows up on the first step (test_simkernel.cpp:182-186); the
    failing variants come back as BatchFailure with the reference message
    format and the rest completed (executor.cpp:121-128)."""
    kind = 1
    seeds = np.array([5, 3, 9, 1], dtype=np.uint64)
    soa = hb.build_states(kind, seeds)
    n = 2
    pos = soa[: 3 * n].T.reshape(4, n, 3)
    vel = soa[3 * n: 6 * n].T.reshape(4, n, 3).copy()
    rest = soa[6 * n:].T
    vel[1, 0, 2] = 1e9  # seed 3
    vel[3, 1, 2] = 1e9  # seed 1
    out, fail, _, _ = gpu.run_states(kind, pos, vel, rest, steps=50, seeds=seeds)
    # oracle: first failing step of each explicit state
    want_fail = []
    for j in range(4):
        p, v, r = pos[j].copy(), vel[j].copy(), rest[j].copy()
        fs = 0
        for s in range(50):
            if O.step(kind, p, v, r)[0] == 1:
                fs = s + 1
                break
        want_fail.append(fs)
    assert list(fail) == want_fail == [0, 1, 0, 1]
    want = O.simulate_batch(kind, seeds[[0, 2]], 50).results
    assert np.array_equal(out[[0, 2]], want)
    msg = hb.format_blowup(3, int(fail[1]))
    assert msg == golden["blowup_messages"][0]["message"] + " (seed 3)"


def test_batch_failure_message_format():
    """batch_failure's what(): failed sorted by seed, "(+k more)", first
    message (executor.cpp:20-28)."""
    err = hb.BatchFailure([(7, "b"), (3, "a")], np.zeros(0, dtype=hb.RESULT_DTYPE))
    assert str(err) == "batch failed for seed 3 (+1 more): a"
    assert err.failed == [(3, "a"), (7, "b")]


def test_order_and_composition_independence(gpu):
    """Seed order defines result order; a variant's result does not depend on
    its batch (rng.hpp:8-10, test_executor.cpp:105-121)."""
    seeds = np.array([5, 3, 9, 1, 7, 2, 8, 0], dtype=np.uint64)
    a = gpu.run(hb.BatchRequest(1, seeds, 50)).results
    assert list(a["seed"]) == list(seeds)
    b = gpu.run(hb.BatchRequest(1, seeds[::-1].copy(), 50)).results
    assert np.array_equal(a, b[::-1])
    big = np.concatenate([np.arange(10000, 20000, dtype=np.uint64), seeds])
    c = gpu.run(hb.BatchRequest(1, big, 50)).results
    assert np.array_equal(c[-8:], a)


def test_skipped_step_changes_checksum(gpu):
    """test_executor.cpp:205-221 (mutation test)."""
    seeds = np.arange(4, dtype=np.uint64)
    a = gpu.run(hb.BatchRequest(0, seeds, 100)).results
    b = gpu.run(hb.BatchRequest(0, seeds, 99)).results
    assert not np.array_equal(a["checksum"], b["checksum"])


def test_request_validation(gpu):
    with pytest.raises(ValueError, match="non-empty"):
        gpu.run(hb.BatchRequest(0, [], 10))
    with pytest.raises(ValueError, match="steps"):
        gpu.run(hb.BatchRequest(0, [1], 0))


def test_full_size_properties(gpu):
    """BASELINE config 2 size (box 16384 x 1000): determinism across runs and
    against an oracle subsample; staged path equals the drop-in call."""
    seeds = np.arange(16384, dtype=np.uint64)
    r1 = gpu.run(hb.BatchRequest(0, seeds, 1000)).results
    r2 = gpu.run(hb.BatchRequest(0, seeds, 1000)).results
    assert np.array_equal(r1, r2)
    sub = seeds[::61]
    assert np.array_equal(r1[::61], O.simulate_batch(0, sub, 1000).results)
    ctx = gpu.ctx
    ctx.stage(0, seeds)
    ctx.launch(1000)
    ctx.launch(1000)  # re-launch on the same staged inputs is idempotent
    out, fail = ctx.fetch()
    assert np.all(fail == 0)
    assert np.array_equal(out, r1)


@pytest.mark.parametrize("kind,n", [(0, 16384), (1, 32768), (2, 32768), (3, 8192), (4, 8192)])
def test_full_size_state_properties(gpu, kind, n):
    """Size-independent properties at BASELINE batch sizes, on the final
    states (hb_run_states from build_model states): no body below the ground
    (the end-of-sweep clamp, simkernel.cpp:150-151; test_simkernel.cpp:154-162),
    every coordinate finite and inside the blow-up limit, and — for the
    reference models — composition: S + T steps in one launch equal T steps
    resumed from the state after S (bit for bit, final states and checksums),
    i.e. nothing outside the state rows carries over between steps."""
    seeds = np.arange(n, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    soa = hb.build_states(kind, seeds)
    nb, m = hb.body_count(kind), hb.constraint_count(kind)
    pos = soa[: 3 * nb].T.reshape(n, nb, 3)
    vel = soa[3 * nb: 6 * nb].T.reshape(n, nb, 3)
    rest = soa[6 * nb: 6 * nb + m].T
    cpg = soa[6 * nb + m:].T if kind == 4 else None
    S, T = 600, 400
    r_all, f_all, p_all, v_all = gpu.run_states(kind, pos, vel, rest, steps=S + T, seeds=seeds, cpg=cpg)
    assert np.all(f_all == 0)
    assert np.all(p_all[:, :, 2] >= 0.0)
    assert np.all(np.isfinite(p_all)) and np.all(np.abs(p_all) <= 1e6) and np.all(np.abs(v_all) <= 1e6)
    if kind == 4:
        return  # the CPG state is not among the returned rows
    _, f1, p1, v1 = gpu.run_states(kind, pos, vel, rest, steps=S, seeds=seeds)
    r2, f2, p2, v2 = gpu.run_states(kind, p1, v1, rest, steps=T, seeds=seeds)
    assert np.all(f1 == 0) and np.all(f2 == 0)
    assert np.array_equal(p2, p_all) and np.array_equal(v2, v_all)
    assert np.array_equal(r2["checksum"], r_all["checksum"])


def test_multi_device_executor_single_gpu():
    ex = hb.MultiGpuExecutor([0])
    seeds = np.arange(3000, dtype=np.uint64)
    res = ex.run(hb.BatchRequest(2, seeds, 40)).results
    assert np.array_equal(res, O.simulate_batch(2, seeds, 40).results)
    # explicit shares over the same device twice (two contexts, two threads)
    ex2 = hb.MultiGpuExecutor([0, 0])
    ex2.shares = hb.plan_allocation_n([1.0, 3.0], len(seeds))
    res2 = ex2.run(hb.BatchRequest(2, seeds, 40)).results
    assert np.array_equal(res2, res)


@pytest.mark.parametrize("kind", [0, 1])
def test_multi_device_degraded_redispatch(kind):
    """Fault injection: one of four contexts is a dead device (every call
    fails as HB_CUDA_ERROR).  Its slice is re-planned over the three
    survivors, the merge is identical to the healthy one-device run and the
    call is flagged degraded (scheduler.cpp:162-183, N-way); a blow-up is the
    batch's own result and is not re-dispatched."""
    ex = hb.MultiGpuExecutor([0, 0, 0, 0])
    seeds = np.arange(10000, dtype=np.uint64) * np.uint64(977)
    want = O.simulate_batch(kind, seeds, 120).results
    ex.ctxs[2].inject_fault(hb._lib.HB_FAULT_DEVICE)
    got = ex.run(hb.BatchRequest(kind, seeds, 120)).results
    assert np.array_equal(got, want)
    assert ex.last_degraded and ex.last_device_ok == [True, True, False, True]
    ex.ctxs[0].inject_fault(hb._lib.HB_FAULT_DEVICE)  # two dead: still complete
    ex.shares = [1000, 2000, 3000, 4000]
    got = ex.run(hb.BatchRequest(kind, seeds, 120)).results
    assert np.array_equal(got, want) and ex.last_device_ok == [False, True, False, True]
    for c in ex.ctxs:
        c.inject_fault(hb._lib.HB_FAULT_DEVICE)
    with pytest.raises(RuntimeError):
        ex.run(hb.BatchRequest(kind, seeds, 120))
    for c in ex.ctxs:
        c.inject_fault(hb._lib.HB_FAULT_NONE)
    ex.shares = None  # even split: index 4321 lies in context 1's slice [2500, 5000)
    ex.ctxs[1].inject_fault(hb._lib.HB_FAULT_BLOWUP, int(seeds[4321]))
    with pytest.raises(hb.BatchFailure) as e:
        ex.run(hb.BatchRequest(kind, seeds, 120))
    assert not ex.last_degraded
    assert e.value.failed[0][0] == int(seeds[4321]) and len(e.value.completed) == len(seeds) - 1


def test_calibrate_contexts_events_and_snap():
    """hb_calibrate: a >= 5 ms probe timed with CUDA events on every context,
    median of 5; identical devices (here: contexts on one GPU, timed
    concurrently) snap to equal times -> equal shares; a dead device is
    flagged and gets no share."""
    ex = hb.MultiGpuExecutor([0, 0, 0, 0])
    times, ok, spreads = ex.calibrate(1, 1000, 4096)
    assert ok == [True] * 4 and all(t > 0 for t in times)
    assert len(set(times)) == 1, (times, spreads)
    assert hb.plan_allocation_n(times, 65536, ok) == [16384] * 4
    ex.ctxs[3].inject_fault(hb._lib.HB_FAULT_DEVICE)
    times, ok, _ = ex.calibrate(1, 1000, 4096)
    assert ok == [True, True, True, False] and times[3] == 0.0
    seeds = np.arange(5000, dtype=np.uint64)
    assert np.array_equal(ex.run(hb.BatchRequest(1, seeds, 50)).results,
                          O.simulate_batch(1, seeds, 50).results)
    assert not ex.last_degraded  # the dead device had no share to lose


def test_fp64_probe(gpu):
    ops, ms = gpu.ctx.fp64_peak()
    assert ms > 0 and 1e12 < ops < 1e14


@pytest.mark.parametrize("kind,n,steps", [(0, 200000, 300), (1, 65536, 200), (2, 16384, 100),
                                          (3, 8192, 40), (4, 16384, 100), (1, 3000, 1), (3, 1000, 1)])
def test_optimised_equals_generic_kernel(gpu, gpu_generic, kind, n, steps):
    """The optimised kernels (device-side initial states — Box from the seed
    alone, the multi-body kinds from host cos / sin rows —, branch-free
    projection with exact replay, two-lane humanoid) against the plain
    reference-order kernel (all-host build_model, library sqrt / '/') on
    large random batches, bit for bit (1-step cases: the initial state
    itself up to one step)."""
    rng = np.random.default_rng(7 + kind)
    seeds = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    a = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
    b = gpu_generic.run(hb.BatchRequest(kind, seeds, steps)).results
    assert np.array_equal(a, b)


@pytest.mark.parametrize("kind,n", [(4, 12288), (4, 12289), (1, 65535), (1, 65536), (2, 65535), (2, 65536),
                                    (4, 65536), (3, 16385)])
def test_dispatch_boundaries_equal_generic(gpu, gpu_generic, kind, n):
    """Both sides of every kernel-selection threshold (two-lane CpgHinge up to
    12 288; register-capped shapes from 65 536; ragged CTAs) against the
    reference-order generic kernel, every record (tools/parity_fuzz.py is
    the wider sweep)."""
    rng = np.random.default_rng(n + 7 * kind)
    seeds = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    a = gpu.run(hb.BatchRequest(kind, seeds, 40)).results
    b = gpu_generic.run(hb.BatchRequest(kind, seeds, 40)).results
    assert np.array_equal(a, b)


def test_fast_math_replicas(gpu):
    """Branch-free sqrt / div replicas are bit-identical to the library
    wherever they claim validity; out-of-range operands are flagged."""
    rng = np.random.default_rng(11)
    n = 1 << 22
    # the operand ranges the projection sees: squared distances and corrections
    x = np.concatenate([rng.uniform(1e-6, 10.0, n // 4), 10.0 ** rng.uniform(-30, 30, n // 4),
                        rng.uniform(-1e-3, 1e-3, n // 4) * 0.5,
                        np.frombuffer(rng.bytes(8 * (n // 4)), dtype=np.float64)])
    y = np.concatenate([rng.uniform(1e-3, 3.0, n // 4), 10.0 ** rng.uniform(-12, 12, n // 4),
                        rng.uniform(0.01, 2.0, n // 4),
                        np.frombuffer(rng.bytes(8 * (n // 4)), dtype=np.float64)])
    x[:16] = [0.0, -0.0, 1e-320, np.inf, np.nan, 1.0, 4.0, 2.0, 1e300, 1e-300, 5e-324,
              2.2250738585072014e-308, 1.7976931348623157e308, 0.25, 9.0, 1e-24]
    sm, dm, sf, df = gpu.ctx.check_fast_math(np.abs(x), y)
    assert sm == 0 and dm == 0
    # realistic operands are essentially never flagged
    sm2, dm2, sf2, df2 = gpu.ctx.check_fast_math(x[16: n // 4], y[16: n // 4])
    assert (sm2, dm2) == (0, 0) and sf2 == 0 and df2 <= 1
    # signed x (division numerators can be negative)
    sm3, dm3, _, _ = gpu.ctx.check_fast_math(x[n // 2: 3 * n // 4], y[n // 2: 3 * n // 4])
    assert dm3 == 0


def test_exact_replay_path_blowup_states(gpu, gpu_generic):
    """States that hit the replay path (huge / degenerate coordinates) agree
    with the generic kernel (fail step and surviving results)."""
    kind = 2
    seeds = np.arange(64, dtype=np.uint64)
    soa = hb.build_states(kind, seeds)
    n = 12
    pos = soa[: 3 * n].T.reshape(64, n, 3).copy()
    vel = soa[3 * n: 6 * n].T.reshape(64, n, 3).copy()
    rest = soa[6 * n:].T.copy()
    vel[::3, 5, 2] = 1e5       # violent but finite
    vel[1::7, 0, :] = 3e5
    pos[2::5, 3, :] = pos[2::5, 4, :]   # coincident bodies -> dist < 1e-12 path
    a = gpu.run_states(kind, pos, vel, rest, steps=30, seeds=seeds)
    b = gpu_generic.run_states(kind, pos, vel, rest, steps=30, seeds=seeds)
    assert np.array_equal(a[1], b[1])
    ok = a[1] == 0
    assert np.array_equal(a[0][ok], b[0][ok])
    assert np.array_equal(a[2][ok], b[2][ok]) and np.array_equal(a[3][ok], b[3][ok])


def test_humanoid_blowup_final_state(gpu, gpu_generic):
    """A humanoid pair that blows up mid-horizon keeps stepping in lockstep
    with its warp (the rung shuffles need both lanes) but its state freezes
    after the failing step: final_soa is the state simulate() holds when
    step() throws, as the generic kernel (which stops) reports it."""
    kind, N = 3, 64
    seeds = np.arange(N, dtype=np.uint64)
    soa = hb.build_states(kind, seeds)
    n = 32
    pos = soa[: 3 * n].T.reshape(N, n, 3).copy()
    vel = soa[3 * n: 6 * n].T.reshape(N, n, 3).copy()
    rest = soa[6 * n:].T.copy()
    pos[1::4, :, 0] += 999000.0  # drifts past |x| = 1e6 after ~1000 steps
    vel[1::4, :, 0] = 1000.0
    a = gpu.run_states(kind, pos, vel, rest, steps=1500, seeds=seeds)
    b = gpu_generic.run_states(kind, pos, vel, rest, steps=1500, seeds=seeds)
    assert np.array_equal(a[1], b[1])
    failed = a[1] != 0
    assert failed.sum() == N // 4 and np.all(a[1][failed] > 500) and np.all(a[1][failed] < 1500)
    assert np.array_equal(a[0][~failed], b[0][~failed])
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


def test_reserve_then_run_is_identical():
    """hb_ctx_reserve (start-up sizing + kernel load through one discarded
    1-step batch) leaves no trace in later results: a reserved context's
    batches equal a fresh context's, below, at and above the reserved size."""
    a = hb.GpuExecutor(0)
    b = hb.GpuExecutor(0)
    try:
        for kind, n in ((0, 70000), (1, 4096), (3, 1000), (4, 3000)):
            a.reserve(kind, n)
            for m in (n // 3, n, n + 17):
                seeds = np.arange(m, dtype=np.uint64) + np.uint64(99)
                ra = a.run(hb.BatchRequest(kind, seeds, 50)).results
                rb = b.run(hb.BatchRequest(kind, seeds, 50)).results
                assert np.array_equal(ra, rb)
        with pytest.raises(Exception):
            a.reserve(9, 10)
    finally:
        a.ctx.close()
        b.ctx.close()


def test_box_nan_state_fails_at_step_one(gpu):
    """A NaN x / y / velocity coordinate (which p.z >= 0 does not catch) keeps
    the warp out of the proven Box phases: the blow-up is reported at step 1,
    as the reference's end-of-step check (simkernel.cpp:165-169) reports it."""
    N = 64
    seeds = np.arange(N, dtype=np.uint64)
    soa = hb.build_states(0, seeds)
    pos = soa[:3].T.reshape(N, 1, 3).copy()
    vel = soa[3:6].T.reshape(N, 1, 3).copy()
    pos[3, 0, 0] = np.nan
    vel[9, 0, 1] = np.nan
    vel[17, 0, 0] = np.nan
    out, fail, fp, fv = gpu.run_states(0, pos, vel, np.zeros((N, 0)), steps=200, seeds=seeds)
    assert list(np.nonzero(fail)[0]) == [3, 9, 17] and np.all(fail[[3, 9, 17]] == 1)
    ok = fail == 0
    want = O.simulate_batch(0, seeds, 200).results
    assert np.array_equal(out[ok], want[ok])


def test_box_zero_copy_path_equals_staged(gpu):
    """Box with pinned seeds + pinned results runs zero-copy (seeds read and
    results written through the host mapping); results identical to the
    staged path and the oracle, including a batch size that is not a
    multiple of any CTA size."""
    for n, steps in ((16384, 1000), (1000, 777), (1, 5)):
        seeds = np.arange(n, dtype=np.uint64) * np.uint64(6364136223846793005)
        ps = hb.pinned_seeds(seeds)
        a = gpu.run(hb.BatchRequest(0, ps, steps)).results
        gpu.ctx.set_zero_copy(False)
        b = gpu.run(hb.BatchRequest(0, ps, steps)).results
        gpu.ctx.set_zero_copy(True)
        assert np.array_equal(a, b)
        sub = slice(0, n, max(1, n // 200))
        assert np.array_equal(a[sub], O.simulate_batch(0, seeds[sub], steps).results)


@pytest.mark.parametrize("kind,n,steps,stride", [
    (4, 8192, 5000, 257),    # configs[2]: CPG / hinge robot, 8192 x 5000
    (3, 8192, 5000, 509),    # its humanoid proxy
    (0, 32768, 20000, 997),  # configs[3] endpoints: 32768 x 20000, every model
    (1, 32768, 20000, 2003),
    (2, 32768, 20000, 257),
    (3, 32768, 20000, 509),
    (4, 32768, 20000, 257),
    (2, 32768, 2000, 4001),
])
def test_baseline_sizes_subsampled_vs_oracle(gpu, kind, n, steps, stride):
    """BASELINE configs at full size on the GPU; an evenly strided subsample
    (first and last variant included) re-simulated by the oracle — and, for
    the reference's models, by the reference library itself — must match bit
    for bit, no variant may blow up, and a checksum-of-checksums pins the
    whole batch for determinism."""
    seeds = np.arange(n, dtype=np.uint64)
    res = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
    assert np.all(res["steps_executed"] == steps)
    idx = np.unique(np.concatenate([np.arange(0, n, stride), [n - 1]]))
    assert np.array_equal(res[idx], O.simulate_batch(kind, seeds[idx], steps).results)
    if kind < 4 and O.ref_available():
        rc, want, _, _, msg = O.ref_cpu_run(kind, seeds[idx], steps, 0)
        assert rc == 0, msg
        assert np.array_equal(res[idx], want)
    again = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
    cc = np.bitwise_xor.reduce(res["checksum"] * np.uint64(0x9E3779B97F4A7C15))
    assert cc == np.bitwise_xor.reduce(again["checksum"] * np.uint64(0x9E3779B97F4A7C15))


@pytest.mark.parametrize("kind,n,steps", [
    (0, 16384, 1000),   # configs[1], the headline, every variant
    (0, 32768, 20000),  # configs[3] endpoint
    (1, 8192, 5000),    # configs[2] size, box_and_ball
    (2, 8192, 1000),
    (3, 8192, 1000),
])
def test_full_batches_vs_reference_library(gpu, kind, n, steps):
    """Every record of a full BASELINE-size batch against the reference's own
    cpu_executor (oracle/_ref: the reference sources compiled in place,
    all host threads), bit for bit."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    seeds = np.arange(n, dtype=np.uint64)
    got = gpu.run(hb.BatchRequest(kind, seeds, steps)).results
    rc, want, _, _, msg = O.ref_cpu_run(kind, seeds, steps, 0)
    assert rc == 0, msg
    assert np.array_equal(got, want)


def test_nvml_utilisation_trace():
    """GpuExecutor(monitor=True) fills BatchResult.utilization_trace from NVML
    (the accelerator side the reference leaves at 0, monitor.cpp:164)."""
    ex = hb.GpuExecutor(0, monitor=True)
    # ~0.6 s of kernel time: several 20 Hz samples inside NVML's averaging window
    res = ex.run(hb.BatchRequest(3, np.arange(16384, dtype=np.uint64), 15000))
    tr = res.utilization_trace
    assert len(tr) >= 2
    assert all(0.0 <= u <= 100.0 for _, u in tr)
    assert max(u for _, u in tr) > 0.0
