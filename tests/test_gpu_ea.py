"""GPU generation loop (hb_run_ea) parity: genomes and fitness of every
generation bit-identical to the reference run_ea (golden) and the oracle."""
import numpy as np
import pytest

import oracle as O
import paper_2502_11129_b200 as hb
from helpers import OracleExecutor

pytestmark = pytest.mark.gpu


def bits(x):
    return "%016x" % int(np.float64(x).view(np.uint64))


def test_native_ea_matches_reference_golden(gpu, golden):
    for g in golden["run_ea"]:
        r = hb.run_ea(g["kind"], g["pop"], g["generations"], g["steps"], gpu, g["seed"])
        assert ["%016x" % int(x) for x in r.population.genomes] == g["genomes"]
        assert [bits(x) for x in r.population.fitnesses] == g["fitness_bits"]


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_native_history_matches_python_loop(gpu, kind):
    pop, gens, steps = (4096, 1024, 256, 128)[kind], 4, (200, 100, 40, 20)[kind]
    nat = hb.run_ea(kind, pop, gens, steps, gpu, seed=5, keep_history=True)
    ref = hb.run_ea(kind, pop, gens, steps, OracleExecutor(8), seed=5, keep_history=True)
    assert len(nat.history) == gens + 1
    for (g1, f1), (g2, f2) in zip(nat.history, ref.history):
        assert np.array_equal(g1, g2)
        assert np.array_equal(f1.view(np.uint64), f2.view(np.uint64))
    assert nat.best_fitness == ref.best_fitness


def test_python_loop_over_gpu_executor_equals_native(gpu):
    a = hb.run_ea(1, 2048, 3, 150, gpu, seed=9, native=False)
    b = hb.run_ea(1, 2048, 3, 150, gpu, seed=9)
    assert np.array_equal(a.population.genomes, b.population.genomes)
    assert np.array_equal(a.population.fitnesses, b.population.fitnesses)


def test_config5_population_box_and_ball():
    """BASELINE config 5 population size (65 536) on one device vs the
    oracle's run_ea (shorter horizon to keep the CPU checker in seconds)."""
    ex = hb.GpuExecutor(0)
    r = hb.run_ea(1, 65536, 2, 60, ex, seed=0)
    g, f = O.run_ea(1, 65536, 2, 60, seed=0)
    assert np.array_equal(r.population.genomes, g)
    assert np.array_equal(r.population.fitnesses, f)
    assert r.profile.evaluation_s > 0


def test_sharded_over_two_contexts(gpu):
    """Two contexts on the same device stand in for two GPUs: offspring are
    split by the N-way splitter and fitness gathered by peer copy."""
    ex = hb.MultiGpuExecutor([0, 0])
    for kind in (0, 2):
        a = hb.run_ea_native(kind, 2000, 3, 50, ex, seed=1, device_times=[1.0, 3.0])
        b = hb.run_ea(kind, 2000, 3, 50, gpu, seed=1)
        assert np.array_equal(a.population.genomes, b.population.genomes)
        assert np.array_equal(a.population.fitnesses, b.population.fitnesses)


def test_native_preconditions(gpu):
    for pop, gens in ((5, 1), (0, 1), (4, 0)):
        with pytest.raises(ValueError):
            hb.run_ea(0, pop, gens, 10, gpu)
