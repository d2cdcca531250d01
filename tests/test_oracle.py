"""The oracle is pinned before it is trusted: the C restatement
(oracle/hb_oracle.c) against the committed golden vectors (generated from the
reference itself) and, when present, against the compiled reference library.
Also restates the reference's own known-answer tests
(proj/tests/test_simkernel.cpp) against the restatement."""
import numpy as np
import pytest

import oracle as O


def bits(x):
    return "%016x" % int(np.float64(x).view(np.uint64))


def test_appendix_a_values():
    # SURVEY.md Appendix A (reference compiled with g++ -O3).
    expect = {
        (0, 0): ("0.78230233101847757", "632f1bc723913715"),
        (0, 1): ("0.88828245637634262", "a015cbd8be46905d"),
        (0, 42): ("0.76023474285360537", "db619739610ab341"),
        (1, 0): ("0.78278079498123354", "1c71d1b7aa006ddb"),
        (2, 1): ("0.87777424644371438", "cf5355918c964a82"),
        (3, 0): ("0.74389934710429451", "431f97586e44c894"),
        (3, 42): ("0.81456294398605988", "2db177a5f88ea172"),
    }
    for (k, s), (fit, cs) in expect.items():
        rc, r, _ = O.simulate(k, s, 1000)
        assert rc == 0
        assert "%.17g" % r[1] == fit
        assert "%016x" % r[2] == cs


def test_oracle_matches_golden_simulate(golden):
    for g in golden["simulate"]:
        rc, r, _ = O.simulate(g["kind"], int(g["seed"]), g["steps"])
        assert rc == 0
        assert bits(r[1]) == g["fitness_bits"], g
        assert "%016x" % r[2] == g["checksum"], g
        assert r[3] == g["steps"]


def test_oracle_matches_golden_c1(golden):
    for g in golden["c1"]:
        rc, r, _ = O.simulate(g["kind"], int(g["seed"]), g["steps"])
        assert (bits(r[1]), "%016x" % r[2]) == (g["fitness_bits"], g["checksum"])


def test_oracle_build_model_golden(golden):
    for g in golden["build_model"]:
        p, v, r = O.build_model(g["kind"], int(g["seed"]))
        assert [bits(x) for x in p.ravel()] == g["pos_bits"]
        assert [bits(x) for x in v.ravel()] == g["vel_bits"]
        assert [bits(x) for x in r] == g["rest_bits"]


def test_oracle_trajectories_golden(golden):
    for g in golden["trajectory"]:
        p, v, r = O.build_model(g["kind"], int(g["seed"]))
        t = 0.0
        for _ in range(g["steps"]):
            rc, t = O.step(g["kind"], p, v, r, O.DT, t)
            assert rc == 0
        assert [bits(x) for x in p.ravel()] == g["pos_bits"]
        assert [bits(x) for x in v.ravel()] == g["vel_bits"]
        assert bits(t) == g["time_bits"]


def test_known_answers(golden):
    ka = golden["known_answers"]
    # rest on the ground (test_simkernel.cpp:106-115)
    p = np.array([[0.3, -0.2, 0.0]]); v = np.zeros((1, 3))
    rc, _ = O.step(0, p, v, np.zeros(0))
    assert rc == 0
    assert [bits(x) for x in p.ravel()] == ka["rest_on_ground"]["pos_bits"]
    assert abs(p[0, 0] - 0.3) < 1e-9 and abs(p[0, 2]) < 1e-9 and v[0, 2] == 0.0
    # free fall (:117-126)
    p = np.array([[0.0, 0.0, 5.0]]); v = np.zeros((1, 3))
    O.step(0, p, v, np.zeros(0))
    expected = -9.81 * O.DT * (1.0 - 0.8 * O.DT)
    assert abs(v[0, 2] - expected) < 1e-12
    assert [bits(x) for x in v.ravel()] == ka["free_fall"]["vel_bits"]
    # blow-up (:182-186)
    p, v, r = O.build_model(0, 0)
    v[0] = [0.0, 0.0, 1e9]
    rc, t = O.step(0, p, v, r)
    assert rc == 1 and ka["blowup_vz_1e9"]["rc"] == 1
    # non-positive dt (:128-132)
    assert O.step(0, p, v, r, 0.0)[0] == -1


def test_blowup_message_format(golden):
    for g in golden["blowup_messages"]:
        msg = O.blowup_message(99, g["fail_step"])
        assert msg == g["message"] + " (seed 99)"


def test_energy_and_ground_properties():
    # test_simkernel.cpp:134-162 on the restatement
    for kind in range(4):
        p, v, r = O.build_model(kind, 2)
        def energy():
            return float(np.sum(0.5 * np.sum(v * v, axis=1) + 9.81 * p[:, 2]))
        e = [energy()]
        for _ in range(300):
            O.step(kind, p, v, r)
            e.append(energy())
            assert p[:, 2].min() >= -1e-6
        for k in range(0, len(e) - 10, 10):
            assert e[k + 10] <= e[k] * (1 + 1e-9) + 1e-12
        assert e[-1] <= e[0]


def test_plan_allocation_golden(golden):
    for g in golden["plan_allocation"]:
        tc = float(np.uint64(int(g["t_cpu_bits"], 16)).view(np.float64))
        ta = float(np.uint64(int(g["t_accel_bits"], 16)).view(np.float64))
        p = O.plan_allocation(tc, ta, g["n"])
        assert (p[1], p[2], bits(p[4])) == (g["n_cpu"], g["n_accel"], g["frac_bits"])
    for g in golden["plan_reference_splits"]:
        p = O.plan_allocation(g["t_cpu"], g["t_accel"], g["n"], g["cpu_ok"], g["accel_ok"])
        assert (p[1], p[2], bits(p[4])) == (g["n_cpu"], g["n_accel"], g["frac_bits"])


def test_run_ea_golden(golden):
    for g in golden["run_ea"]:
        gen, fit = O.run_ea(g["kind"], g["pop"], g["generations"], g["steps"], g["seed"], threads=2)
        assert ["%016x" % int(x) for x in gen] == g["genomes"]
        assert [bits(x) for x in fit] == g["fitness_bits"]


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_restatement_equals_reference_random_seeds():
    rng = np.random.default_rng(0)
    seeds = rng.integers(0, 2**63, size=600, dtype=np.uint64)
    for kind in range(4):
        steps = (400, 200, 60, 30)[kind]
        a = O.simulate_batch(kind, seeds, steps, threads=4)
        rc, b, _, _, _ = O.ref_cpu_run(kind, seeds, steps, workers=4)
        assert rc == 0
        assert np.array_equal(a.results, b)


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_restatement_plan_equals_reference():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        tc, ta = rng.uniform(1e-6, 10, 2)
        n = int(rng.integers(1, 100000))
        assert O.plan_allocation(tc, ta, n) == O.ref_plan_allocation(tc, ta, n)
