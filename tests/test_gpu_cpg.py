"""CpgHinge on the GPU vs its defining oracle (the reference has no such
model; parity is against oracle/hb_oracle.c).  Bit-exact."""
import numpy as np
import pytest

import oracle as O
import paper_2502_11129_b200 as hb
from helpers import OracleExecutor

pytestmark = pytest.mark.gpu


def test_random_batches_vs_oracle(gpu):
    seeds = np.random.default_rng(44).integers(0, 2**64 - 1, 1024, dtype=np.uint64, endpoint=True)
    for steps in (1, 37, 500):
        got = gpu.run(hb.BatchRequest(4, seeds, steps)).results
        want = O.simulate_batch(4, seeds, steps)
        assert np.all(want.fail_step == 0)
        assert np.array_equal(got, want.results), steps


def test_long_horizon_config3_steps(gpu):
    seeds = np.arange(64, dtype=np.uint64) * np.uint64(31337)
    got = gpu.run(hb.BatchRequest(4, seeds, 5000)).results
    assert np.array_equal(got, O.simulate_batch(4, seeds, 5000).results)


def test_optimised_equals_generic():
    a = hb.GpuExecutor(0)
    b = hb.GpuExecutor(0, kernel=1)
    seeds = np.random.default_rng(5).integers(0, 2**63, 32768, dtype=np.uint64)
    ra = a.run(hb.BatchRequest(4, seeds, 100)).results
    rb = b.run(hb.BatchRequest(4, seeds, 100)).results
    assert np.array_equal(ra, rb)


def test_zero_cpg_is_the_passive_robot(gpu):
    """Known answer: zero CPG parameters -> the passive robot (oracle step
    without actuation), including the final state, bit for bit."""
    seeds = np.arange(16, dtype=np.uint64)
    soa = hb.build_states(4, seeds)
    pos = soa[:27].T.reshape(16, 9, 3)
    vel = soa[27:54].T.reshape(16, 9, 3)
    rest = soa[54:66].T
    cpg = np.zeros((16, 16))
    out, fail, fp, fv = gpu.run_states(4, pos, vel, rest, steps=200, seeds=seeds, cpg=cpg)
    assert np.all(fail == 0)
    for j in range(16):
        p, v, r = pos[j].copy(), vel[j].copy(), rest[j].copy()
        for _ in range(200):
            assert O.step(4, p, v, r)[0] == 0
        assert np.array_equal(fp[j].view(np.uint64), p.view(np.uint64))
        assert np.array_equal(fv[j].view(np.uint64), v.view(np.uint64))


def test_ea_controller_evolution(gpu):
    """Controller evolution: the genome seeds the CPG parameters; the native
    loop matches the oracle-backed loop generation by generation."""
    a = hb.run_ea(4, 512, 3, 200, gpu, seed=2, keep_history=True)
    b = hb.run_ea(4, 512, 3, 200, OracleExecutor(8), seed=2, keep_history=True)
    for (g1, f1), (g2, f2) in zip(a.history, b.history):
        assert np.array_equal(g1, g2) and np.array_equal(f1, f2)


def _cpg_states(N, seed=0):
    seeds = np.arange(N, dtype=np.uint64) + np.uint64(seed)
    soa = hb.build_states(4, seeds)
    pos = soa[:27].T.reshape(N, 9, 3).copy()
    vel = soa[27:54].T.reshape(N, 9, 3).copy()
    rest = soa[54:66].T.copy()
    cpg = soa[66:82].T.copy()
    return seeds, pos, vel, rest, cpg


@pytest.mark.parametrize("n", [1, 3, 31, 33, 1000, 8192])
def test_pair_kernel_sizes_vs_oracle(gpu, n):
    """The two-lane latency kernel (n <= 12 288) at ragged sizes: partial
    warps and CTAs, a lone pair; every record against the oracle."""
    seeds = np.random.default_rng(n).integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    assert hb.kernel_name(4, n) == "cpg_pair_kernel"
    got = gpu.run(hb.BatchRequest(4, seeds, 120)).results
    assert np.array_equal(got, O.simulate_batch(4, seeds, 120).results)


def test_pair_kernel_blowup_and_replay_states(gpu, gpu_generic):
    """Two-lane kernel against the generic kernel from crafted states: pairs
    that blow up at different steps (their state freezes while the warp keeps
    stepping), coincident bodies (dist < 1e-12: the exact replay), violent
    velocities; fail steps, results and final states identical."""
    N = 96
    seeds, pos, vel, rest, cpg = _cpg_states(N)
    pos[1::4, :, 0] += 999000.0     # drift past |x| = 1e6 mid-horizon
    vel[1::4, :, 0] = 1000.0 + np.arange(len(vel[1::4]))[:, None]
    pos[2::5, 2, :] = pos[2::5, 1, :]  # hinge-tip link of limb 0 degenerate
    pos[3::7, 0, :] = pos[3::7, 8, :]  # core on tip 3 (an actuated link)
    vel[5::9, 4, 2] = 2e5
    a = gpu.run_states(4, pos, vel, rest, steps=1500, seeds=seeds, cpg=cpg)
    b = gpu_generic.run_states(4, pos, vel, rest, steps=1500, seeds=seeds, cpg=cpg)
    assert np.array_equal(a[1], b[1])
    assert np.count_nonzero(a[1]) >= N // 4
    ok = a[1] == 0
    assert np.array_equal(a[0][ok], b[0][ok])
    assert np.array_equal(a[2].view(np.uint64), b[2].view(np.uint64))
    assert np.array_equal(a[3].view(np.uint64), b[3].view(np.uint64))


def test_pair_kernel_other_dt(gpu, gpu_generic):
    """dt != 0.002: half_k is then not a power of two and the latency kernel's
    folded division does not apply — every step takes the exact path; still
    bit-identical to the generic kernel."""
    N = 64
    seeds, pos, vel, rest, cpg = _cpg_states(N, 7)
    for dt in (0.0015, 0.001):
        a = gpu.run_states(4, pos, vel, rest, steps=200, dt=dt, seeds=seeds, cpg=cpg)
        b = gpu_generic.run_states(4, pos, vel, rest, steps=200, dt=dt, seeds=seeds, cpg=cpg)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])
        assert np.array_equal(a[2].view(np.uint64), b[2].view(np.uint64))
