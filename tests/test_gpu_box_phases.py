"""Box kernel phase specialisation (airborne / grounded chunks) on explicit
initial states chosen to sit on every phase boundary: exactly grounded
(+0/-0 heights and velocities), heights just above and below the airborne
proof's margin, upward launches that come back down, tall drops, states that
blow up mid-horizon, and time steps outside the fast range.  Every variant's
fail step, final state, fitness and checksum must equal the oracle's
reference-order stepping (oracle/hb_oracle.c, simkernel.cpp:122-170) bit for
bit."""
import numpy as np
import pytest

import oracle as O
import paper_2502_11129_b200 as hb

pytestmark = pytest.mark.gpu


def _edge_states(n, rng):
    seeds = np.arange(n, dtype=np.uint64) + np.uint64(1000)
    soa = hb.build_states(0, seeds)
    pos = soa[:3].T.reshape(n, 1, 3).copy()
    vel = soa[3:6].T.reshape(n, 1, 3).copy()
    g = np.arange(n) % 12
    z, vz = pos[:, 0, 2], vel[:, 0, 2]
    z[g == 0], vz[g == 0] = 0.0, 0.0                       # grounded fixed point
    z[g == 1], vz[g == 1] = -0.0, -0.0                     # signed zeros
    z[g == 2], vz[g == 2] = 0.0, -0.0
    sel = g == 3                                           # around the airborne margin
    vz[sel] = rng.uniform(-8, 8, sel.sum())
    z[sel] = 0.002 * (16.01 * np.abs(vz[sel]) + 121 * 9.81 * 0.002 + 1e-3) * rng.uniform(0.9, 1.1, sel.sum())
    sel = g == 4                                           # tiny heights
    z[sel] = rng.choice([1e-9, 1e-300, 5e-324, 1e-12, 3e-5], sel.sum())
    vz[sel] = rng.uniform(-1, 1, sel.sum())
    sel = g == 5                                           # upward launches
    vz[sel] = rng.uniform(1, 12, sel.sum())
    sel = g == 6                                           # tall drops
    z[sel] = rng.uniform(10, 1e4, sel.sum())
    sel = g == 7                                           # blow-up mid-horizon
    z[sel] = 9.99e5
    vz[sel] = rng.uniform(500, 3000, sel.sum())
    sel = g == 8                                           # large lateral speed
    vel[sel, 0, 0] = rng.uniform(-1e6, 1e6, sel.sum())
    sel = g == 9                                           # below ground, moving
    z[sel] = -rng.uniform(1e-6, 1.0, sel.sum())
    vz[sel] = rng.uniform(-3, 3, sel.sum())
    sel = g == 10                                          # resting, tiny velocity
    z[sel] = 0.0
    vz[sel] = rng.choice([1e-300, -1e-300, 5e-324, 1e-3], sel.sum())
    return seeds, pos, vel


def _air_bound(vz, dt):
    """The kernel's 16-step airborne threshold (box_kernel, airborne proof)."""
    gdt = 9.81 * dt
    return dt * (1.0 + 1e-4) * (16.0 * np.abs(vz) + 136.0 * (gdt + 1e-5)) + 2e-8


def _warp_blocks(dt, rng):
    """Whole warps (32 lanes) that enter a specialised chunk at step 0."""
    w = 32
    pos = np.zeros((4 * w, 1, 3))
    vel = np.zeros((4 * w, 1, 3))
    pos[:, 0, :2] = rng.uniform(-1, 1, (4 * w, 2))
    vel[:, 0, :2] = rng.uniform(-1, 1, (4 * w, 2))
    vz = rng.uniform(-8, 2, w)                      # just above the airborne bound
    vel[:w, 0, 2] = vz
    pos[:w, 0, 2] = _air_bound(vz, dt) * (1 + 1e-12)
    # just above an earlier, too small bound (it omitted the first step's
    # g dt): these land inside the chunk, so an airborne chunk would be wrong
    vz = rng.uniform(-8, 0, w)
    vel[w:2 * w, 0, 2] = vz
    pos[w:2 * w, 0, 2] = (dt * (16.01 * np.abs(vz) + 121.0 * 9.81 * dt + 1e-3) + 1e-8) * (1 + 1e-6)
    pos[2 * w:3 * w, 0, 0] = rng.uniform(9.0e5, 9.6e5, w) * rng.choice([-1, 1], w)
    vel[2 * w:3 * w, 0, 0] = rng.uniform(1e4, 4e5, w) * rng.choice([-1, 1], w)   # grounded, drifts to blow-up
    vel[3 * w:, 0, :2] = rng.uniform(-50, 50, (w, 2))                             # grounded, long run
    return np.arange(4 * w, dtype=np.uint64) + np.uint64(77), pos, vel


def _oracle(pos, vel, steps, dt):
    n = pos.shape[0]
    fail = np.zeros(n, dtype=np.uint64)
    fp, fv = pos.copy(), vel.copy()
    rest = np.zeros(0)
    for j in range(n):
        p, v = fp[j], fv[j]
        t = 0.0
        for s in range(steps):
            rc, t = O.step(0, p, v, rest, dt=dt, time=t)
            if rc == 1:
                fail[j] = s + 1
                break
    return fail, fp, fv


@pytest.mark.parametrize("dt,steps", [(0.002, 1000), (0.002, 37), (0.0025, 300), (1e-4, 200),
                                      (0.01, 300), (2e-5, 100)])
def test_box_phases_edge_states(gpu, dt, steps):
    rng = np.random.default_rng(int(dt * 1e6) + steps)
    seeds, pos, vel = _edge_states(608, rng)
    s2, p2, v2 = _warp_blocks(dt, rng)
    seeds, pos, vel = np.concatenate([seeds, s2]), np.concatenate([pos, p2]), np.concatenate([vel, v2])
    n = len(seeds)
    out, fail, fp, fv = gpu.run_states(0, pos, vel, np.zeros((n, 0)), steps=steps, dt=dt, seeds=seeds)
    want_fail, wp, wv = _oracle(pos, vel, steps, dt)
    assert np.array_equal(fail, want_fail)
    assert np.array_equal(fp.view(np.uint64), wp.view(np.uint64))
    assert np.array_equal(fv.view(np.uint64), wv.view(np.uint64))
    ok = fail == 0
    for j in np.nonzero(ok)[0][:: 7]:
        dx = wp[j, 0, 0] - pos[j, 0, 0]
        dy = wp[j, 0, 1] - pos[j, 0, 1]
        assert out[j]["fitness"] == np.sqrt(dx * dx + dy * dy)
        assert int(out[j]["checksum"]) == O.checksum(wp[j], wv[j])
    if dt == 0.002 and steps == 1000:
        assert (~ok).sum() > 0 and ok.sum() > 0


def test_box_phases_partial_warp(gpu):
    """Batch sizes that leave idle lanes in the last warp."""
    for n in (1, 31, 33, 16383):
        seeds = np.arange(n, dtype=np.uint64) * np.uint64(977)
        got = gpu.run(hb.BatchRequest(0, seeds, 500)).results
        sub = slice(0, n, max(1, n // 150))
        assert np.array_equal(got[sub], O.simulate_batch(0, seeds[sub], 500).results)


def test_box_work_counter(gpu):
    """hb_work_counter: 16 algorithmic ops per variant-step, 10 for steps a
    warp runs at the grounded fixed point; other models do not count."""
    n, steps = 64, 1000
    pos = np.zeros((n, 1, 3))
    vel = np.zeros((n, 1, 3))
    vel[:, 0, :2] = 0.25
    c0 = gpu.ctx.work_counter()
    gpu.run_states(0, pos, vel, np.zeros((n, 0)), steps=steps)
    grounded = (steps // 16) * 16  # the horizon's whole chunks; the 8-step tail runs step()
    assert gpu.ctx.work_counter() - c0 == n * (16 * steps - 6 * grounded)
    c1 = gpu.ctx.work_counter()
    gpu.run(hb.BatchRequest(1, np.arange(32, dtype=np.uint64), 100))
    assert gpu.ctx.work_counter() == c1
    seeds = np.arange(4096, dtype=np.uint64)
    gpu.run(hb.BatchRequest(0, seeds, steps))
    ops = gpu.ctx.work_counter() - c1
    assert 10 * 4096 * steps < ops < 16 * 4096 * steps
