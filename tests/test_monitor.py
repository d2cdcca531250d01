"""monitor.py mirrors proj/src/monitor.cpp (summarize, knee) — checked against
the reference's own test cases (proj/tests/test_monitor.cpp) and, when built,
against the reference library."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_2502_11129_b200 as hb


def test_t_table():
    assert abs(hb.monitor.student_t_critical_95(2) - 4.303) < 1e-3
    assert abs(hb.monitor.student_t_critical_95(30) - 2.042) < 1e-3
    assert hb.monitor.student_t_critical_95(0) == 0.0


def test_summarize():
    s = hb.summarize([1.0, 2.0, 3.0])
    assert s.mean == 2.0 and abs(s.stddev - 1.0) < 1e-15
    assert abs((s.ci95_high - s.mean) - 4.302652729911275 / np.sqrt(3)) < 1e-9
    assert s.small_sample()
    one = hb.summarize([5.0])
    assert one.ci95_low == one.ci95_high == 5.0
    with pytest.raises(ValueError):
        hb.summarize([])


def test_knee_regimes():
    law = [(n, 0.5 + 0.1 * -(-n // 1024)) for n in (32, 128, 256, 512, 1024, 2048, 4096)]
    assert hb.detect_saturation_knee(law) == (1024, hb.KneeRegime.Knee)
    flat = [(n, 1.0) for n in (1, 2, 3)]
    assert hb.detect_saturation_knee(flat) == (3, hb.KneeRegime.AllFlat)
    lin = [(n, float(n)) for n in (1, 2, 3)]
    assert hb.detect_saturation_knee(lin) == (1, hb.KneeRegime.AllLinear)
    with pytest.raises(ValueError):
        hb.detect_saturation_knee([(1, 1.0), (2, 1.0)])
    with pytest.raises(ValueError):
        hb.detect_saturation_knee([(1, 1.0), (1, 1.0), (2, 1.0)])


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_knee_matches_reference_library():
    rng = np.random.default_rng(0)
    for _ in range(300):
        k = int(rng.integers(3, 12))
        ns = np.cumsum(rng.integers(1, 5000, k)).astype(np.uint64)
        walls = rng.uniform(0.1, 2.0, k) if rng.uniform() < 0.5 else np.sort(rng.uniform(0.1, 2.0, k))
        kn, reg = C.c_uint64(0), C.c_int(0)
        O.ref().hbref_detect_knee(ns.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  walls.ctypes.data_as(C.POINTER(C.c_double)), k, 0.05,
                                  C.byref(kn), C.byref(reg))
        n, regime = hb.detect_saturation_knee(list(zip(ns.tolist(), walls.tolist())))
        assert (n, regime.value) == (kn.value, reg.value)


def test_util_sampler_degrades_without_nvml():
    s = hb.GpuUtilSampler(0)
    s.start()
    tr = s.stop()
    assert isinstance(tr, list)
