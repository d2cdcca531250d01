"""CpgHinge — the CPG / hinge modular robot of BASELINE config 3.  The
reference has no such model, so it is DEFINED by the oracle
(oracle/hb_oracle.c, hbo_cpg_*) and everything here is parity against that
definition ("parity unpinned" by the reference).  CPU tests: the oracle's
own properties and the product's host initialiser."""
import json
import os

import numpy as np

import oracle as O
import paper_2502_11129_b200 as hb

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cpg_golden.json")


def bits(x):
    return "%016x" % int(np.float64(x).view(np.uint64))


def test_zero_cpg_reduces_to_passive_robot():
    """omega = c = x(0) = 0 keeps every actuated rest length at L0, so the
    CPG step equals the plain reference step on the same topology, bit for bit."""
    for seed in (0, 1, 99):
        p, v, r, c = O.cpg_build(seed)
        c[:] = 0.0
        p2, v2 = p.copy(), v.copy()
        t1 = t2 = 0.0
        for _ in range(300):
            rc1, t1 = O.cpg_step(p, v, r, c, O.DT, t1)
            rc2, t2 = O.step(4, p2, v2, r, O.DT, t2)
            assert rc1 == rc2 == 0
        assert np.array_equal(p.view(np.uint64), p2.view(np.uint64))
        assert np.array_equal(v.view(np.uint64), v2.view(np.uint64))
        assert np.all(c == 0.0)


def test_cpg_actuation_changes_the_trajectory():
    p, v, r, c = O.cpg_build(3)
    p0, v0, r0, c0 = O.cpg_build(3)
    c0[:] = 0.0
    for _ in range(200):
        O.cpg_step(p, v, r, c)
        O.cpg_step(p0, v0, r0, c0)
    assert not np.array_equal(p, p0)


def test_cpg_stable_and_bounded():
    b = O.simulate_batch(4, np.arange(400, dtype=np.uint64), 3000)
    assert np.all(b.fail_step == 0)
    assert np.all(np.isfinite(b.results["fitness"]))


def test_topology_and_initial_geometry():
    ca = np.zeros(46, dtype=np.int32); cb = np.zeros(46, dtype=np.int32); st = np.zeros(46)
    import ctypes as C
    m = O.lib().hbo_topology(4, ca.ctypes.data_as(C.POINTER(C.c_int)),
                             cb.ctypes.data_as(C.POINTER(C.c_int)),
                             st.ctypes.data_as(C.POINTER(C.c_double)))
    assert m == 12
    assert list(zip(ca[:12], cb[:12])) == [(0, 1), (1, 2), (0, 3), (3, 4), (0, 5), (5, 6), (0, 7),
                                           (7, 8), (0, 2), (0, 4), (0, 6), (0, 8)]
    assert list(st[:8]) == [2.5e5] * 8 and list(st[8:12]) == [1.25e5] * 4
    p, v, r, c = O.cpg_build(7)
    assert np.all(v[:, 2] == 0.0) and np.all(v[:, 0] == v[0, 0])
    assert np.all((c[8:12] >= 2 * np.pi * 0.5) & (c[8:12] < 2 * np.pi * 2.0))
    assert np.all(np.abs(c[12:16]) <= 0.5) and np.all(np.abs(c[0:4]) <= 0.1)


def test_host_initialiser_matches_oracle():
    seeds = np.random.default_rng(1).integers(0, 2**63, 1500, dtype=np.uint64)
    soa = hb.build_states(4, seeds)
    for j in range(0, len(seeds), 5):
        p, v, r, c = O.cpg_build(int(seeds[j]))
        ref = np.concatenate([p.ravel(), v.ravel(), r, c])
        assert np.array_equal(ref.view(np.uint64), soa[:, j].copy().view(np.uint64))


def test_golden_self_consistency():
    """The committed golden values (generated from the oracle by
    tests/golden/make_golden.py) still hold — a change to the model
    definition must be deliberate."""
    g = json.load(open(GOLD))
    for row in g["simulate"]:
        rc, r, _ = O.simulate(4, int(row["seed"]), row["steps"])
        assert rc == 0 and bits(r[1]) == row["fitness_bits"] and "%016x" % r[2] == row["checksum"]
