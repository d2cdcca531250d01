"""Generation loop (ea.cpp:33-145): the Python loop over a CPU back-end
against the reference run_ea golden trajectories, plus the reference's own
EA unit tests (proj/tests/test_ea.cpp)."""
import numpy as np
import pytest

import oracle as O
import paper_2502_11129_b200 as hb
from helpers import FailingExecutor, OracleExecutor


def bits(x):
    return "%016x" % int(np.float64(x).view(np.uint64))


def test_rng_vectorised_matches_reference():
    keys = np.array([0, 1, 2**63, 2**64 - 1, 0xACC1], dtype=np.uint64)
    for k in keys:
        ctr = np.arange(100, dtype=np.uint64) * np.uint64(977)
        got = hb.rng_at(k, ctr)
        assert [int(x) for x in got] == [O.rng_at(int(k), int(c)) for c in ctr]


def test_stable_order_matches_restatement():
    rng = np.random.default_rng(0)
    f = np.round(rng.uniform(0, 1, 5000), 2)  # many exact ties
    assert np.array_equal(hb.stable_order_desc(f), O.stable_order_desc(f))


def test_python_loop_matches_reference_golden(golden):
    ex = OracleExecutor()
    for g in golden["run_ea"]:
        r = hb.run_ea(g["kind"], g["pop"], g["generations"], g["steps"], ex, g["seed"])
        assert ["%016x" % int(x) for x in r.population.genomes] == g["genomes"]
        assert [bits(x) for x in r.population.fitnesses] == g["fitness_bits"]
        assert r.population.generation == g["generations"]


def test_population_cardinality():
    r = hb.run_ea(0, 4, 1, 10, OracleExecutor())
    assert len(r.population.genomes) == 4 and len(r.population.fitnesses) == 4
    assert r.population.generation == 1
    assert r.best_fitness == r.population.fitnesses.max()


def test_preconditions():
    ex = OracleExecutor()
    for pop, gens in ((5, 1), (0, 1), (1, 1), (4, 0)):
        with pytest.raises(ValueError):
            hb.run_ea(0, pop, gens, 10, ex)


def test_pure_function_of_arguments():
    ex = OracleExecutor()
    a = hb.run_ea(1, 8, 3, 25, ex, 42)
    b = hb.run_ea(1, 8, 3, 25, ex, 42)
    assert np.array_equal(a.population.genomes, b.population.genomes)
    assert np.array_equal(a.population.fitnesses, b.population.fitnesses)
    c = hb.run_ea(1, 8, 3, 25, ex, 43)
    assert not np.array_equal(a.population.genomes, c.population.genomes)


def test_elitism_best_non_decreasing():
    ex = OracleExecutor()
    r = hb.run_ea(0, 8, 6, 40, ex, 7, keep_history=True)
    bests = [f.max() for _, f in r.history]
    assert all(b2 >= b1 for b1, b2 in zip(bests, bests[1:]))


def test_phase_accounting():
    r = hb.run_ea(0, 8, 4, 60, OracleExecutor())
    p = r.profile
    acc = p.selection_s + p.variation_s + p.evaluation_s + p.bookkeeping_s
    assert p.evaluation_s > 0 and p.total_s > 0
    assert p.total_s * 0.95 <= acc <= p.total_s * 1.05
    assert 0.0 <= p.evaluation_fraction() <= 1.0


def test_executor_failure_propagates():
    with pytest.raises(RuntimeError):
        hb.run_ea(0, 4, 1, 10, FailingExecutor())


def test_report_profile_format():
    p = hb.PhaseProfile(selection_s=1.0, variation_s=0.5, evaluation_s=8.0, bookkeeping_s=0.5,
                        total_s=10.0)
    lines = hb.report_profile(p).splitlines()
    assert lines[0].startswith("phase")
    assert lines[1].startswith("evaluation") and "0.800" in lines[1]
    assert lines[2].startswith("selection")
    assert lines[3].startswith("variation") and lines[4].startswith("bookkeeping")
    assert lines[5].startswith("total") and "1.000" in lines[5]
    text = hb.report_profile(p)
    assert "profile.evaluation_s=8\n" in text and "profile.total_s=10\n" in text
    assert "profile.evaluation_fraction=0.8\n" in text
    z = hb.report_profile(hb.PhaseProfile())
    assert "0.000" in z and "profile.evaluation_fraction=0\n" in z
    assert "nan" not in z and "inf" not in z
