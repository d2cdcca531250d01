"""CPU-side checks of the product's native library (no compute on a GPU):
it loads, exports every symbol include/hbgpu.h declares, its host-side
initialiser is bit-exact with build_model, and its splitter is bit-exact with
plan_allocation.  On a host without a device, context creation fails loudly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2502_11129_b200 as hb
from paper_2502_11129_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "hbgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert sorted(_lib.EXPORTED) == declared


def test_abi_version_and_model_tables():
    L = _lib.lib
    assert L.hb_abi_version() == 2
    assert [L.hb_body_count(k) for k in range(5)] == [1, 2, 12, 32, 9]
    assert [L.hb_constraint_count(k) for k in range(5)] == [0, 1, 11, 46, 12]
    assert [L.hb_state_rows(k) for k in range(5)] == [6, 13, 83, 238, 82]
    assert L.hb_body_count(5) == -1
    assert [hb.parse_model_kind(hb.to_string(k)) for k in hb.ALL_MODELS] == list(hb.ALL_MODELS)
    with pytest.raises(ValueError):
        hb.parse_model_kind("sphere")


def test_result_struct_layout():
    assert _lib.RESULT_DTYPE.itemsize == 32
    assert list(_lib.RESULT_DTYPE.names) == ["seed", "fitness", "checksum", "steps_executed"]


def test_host_initialiser_bit_exact_golden(golden):
    for g in golden["build_model"]:
        soa = hb.build_states(g["kind"], [int(g["seed"])])[:, 0]
        n, m = O.BODIES[g["kind"]], O.CONSTRAINTS[g["kind"]]
        got = ["%016x" % int(x) for x in soa.view(np.uint64)]
        assert got[: 3 * n] == g["pos_bits"]
        assert got[3 * n: 6 * n] == g["vel_bits"]
        assert got[6 * n:] == g["rest_bits"]


def test_host_initialiser_bit_exact_random():
    rng = np.random.default_rng(5)
    seeds = rng.integers(0, 2**64 - 1, size=2000, dtype=np.uint64)
    for kind in range(4):
        soa = hb.build_states(kind, seeds)
        for j in range(0, len(seeds), 7):
            p, v, r = O.build_model(kind, int(seeds[j]))
            ref = np.concatenate([p.ravel(), v.ravel(), r])
            assert np.array_equal(ref.view(np.uint64), soa[:, j].copy().view(np.uint64))


def test_plan_allocation_bit_exact(golden):
    def bits(x):
        return "%016x" % int(np.float64(x).view(np.uint64))
    for g in golden["plan_allocation"]:
        tc = float(np.uint64(int(g["t_cpu_bits"], 16)).view(np.float64))
        ta = float(np.uint64(int(g["t_accel_bits"], 16)).view(np.float64))
        p = hb.plan_allocation(hb.CalibrationProfile(t_cpu_s=tc, t_accel_s=ta), g["n"])
        assert (p.n_cpu, p.n_accel, bits(p.requested_accel_fraction)) == \
            (g["n_cpu"], g["n_accel"], g["frac_bits"])
        assert p.n_cpu + p.n_accel == g["n"]
    for g in golden["plan_reference_splits"]:
        p = hb.plan_allocation(hb.CalibrationProfile(t_cpu_s=g["t_cpu"], t_accel_s=g["t_accel"],
                                                     cpu_ok=bool(g["cpu_ok"]),
                                                     accel_ok=bool(g["accel_ok"])), g["n"])
        assert (p.n_cpu, p.n_accel) == (g["n_cpu"], g["n_accel"])
    with pytest.raises(ValueError):
        hb.plan_allocation(hb.CalibrationProfile(t_cpu_s=1, t_accel_s=1), 0)


def test_plan_allocation_invariants_random():
    # test_scheduler.cpp:155-177
    rng = np.random.default_rng(2)
    for _ in range(1000):
        tc, ta = rng.uniform(0.1, 10.0, 2)
        n = int(1 + rng.uniform() * 4999.0)
        p = hb.plan_allocation(hb.CalibrationProfile(t_cpu_s=tc, t_accel_s=ta), n)
        assert p.n_cpu + p.n_accel == n
        assert p.accel_fraction == p.n_accel / n
        assert p.requested_accel_fraction == tc / (tc + ta)
        assert abs(p.accel_fraction - p.requested_accel_fraction) * n <= 1.0 + 1e-9
        assert (p.n_total, p.n_cpu, p.n_accel, p.accel_fraction, p.requested_accel_fraction) == \
            O.plan_allocation(tc, ta, n)


def test_nway_plan_reduces_to_two_way():
    rng = np.random.default_rng(3)
    for _ in range(1000):
        tc, ta = rng.uniform(1e-6, 10.0, 2)
        n = int(rng.integers(1, 10001))
        p = hb.plan_allocation(hb.CalibrationProfile(t_cpu_s=tc, t_accel_s=ta), n)
        assert hb.plan_allocation_n([tc, ta], n) == [p.n_cpu, p.n_accel]
    # failed back-ends get nothing; the survivor takes all
    assert hb.plan_allocation_n([1.0, 2.0], 10, ok=[False, True]) == [0, 10]
    assert hb.plan_allocation_n([1.0, 2.0], 10, ok=[True, False]) == [10, 0]


def test_nway_plan_properties():
    rng = np.random.default_rng(4)
    for _ in range(300):
        cnt = int(rng.integers(2, 9))
        t = rng.uniform(0.05, 5.0, cnt)
        n = int(rng.integers(1, 200000))
        sh = hb.plan_allocation_n(list(t), n)
        assert sum(sh) == n and min(sh) >= 0
        # proportional to throughput within rounding (±1 per peel)
        ideal = (1.0 / t) / np.sum(1.0 / t) * n
        assert np.all(np.abs(np.array(sh) - ideal) <= cnt + 1e-9)
    # equal GPUs split evenly (within one variant per peel)
    sh = hb.plan_allocation_n([1.0] * 8, 65536)
    assert sh == [8192] * 8
    ok = [True, False, True, True]
    sh = hb.plan_allocation_n([1.0, 1.0, 1.0, 1.0], 99, ok=ok)
    assert sh[1] == 0 and sum(sh) == 99


def test_plan_allocation_optimal_reference_cases():
    lin = float
    p = hb.plan_allocation_optimal(lin, lin, 100)
    assert (p.n_cpu, p.n_accel) == (50, 50)
    p = hb.plan_allocation_optimal(lin, lin, 101)
    assert (p.n_cpu, p.n_accel) == (51, 50)


def test_format_blowup_matches_reference_text(golden):
    for g in golden["blowup_messages"]:
        assert hb.format_blowup(7, g["fail_step"]) == g["message"] + " (seed 7)"
        assert hb.format_blowup(7, g["fail_step"]) == O.blowup_message(7, g["fail_step"])


def test_no_device_fails_loudly():
    if hb.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(RuntimeError, match="hb_ctx_create"):
        hb.GpuExecutor(0)
    h = C.c_void_p()
    assert _lib.lib.hb_ctx_create(0, C.byref(h)) == _lib.HB_NO_DEVICE


def test_product_does_not_import_oracle():
    """The product never imports, links or calls the checker (comments may
    cite the oracle's definitions)."""
    pkg = os.path.join(ROOT, "paper_2502_11129_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            path = os.path.join(dirpath, f)
            if f.endswith(".py"):
                src = open(path).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "libhboracle" not in src and "libhetbench_ref" not in src, f
            elif f.endswith((".cpp", ".cu", ".h", ".hpp")):
                src = open(path).read()
                code = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
                code = re.sub(r"//[^\n]*", "", code)
                assert "hb_oracle" not in code and "hbo_" not in code, f
                assert "hetbench/" not in code, f  # no reference headers either


def test_model_kind_enum_matches_header():
    """hb_model_kind in include/hbgpu.h carries every kind the runtime
    accepts, CpgHinge (4) included, with the Python ordinals."""
    import re
    with open(os.path.join(ROOT, "include", "hbgpu.h")) as f:
        text = f.read()
    enum = dict((n, int(v)) for n, v in re.findall(r"HB_(BOX|BOX_AND_BALL|ARM_WITH_ROPE|HUMANOID|CPG_HINGE) = (\d)",
                                                   text))
    assert enum == {"BOX": 0, "BOX_AND_BALL": 1, "ARM_WITH_ROPE": 2, "HUMANOID": 3, "CPG_HINGE": 4}
    assert [int(k) for k in hb.ALL_MODELS] == sorted(enum.values())


def test_snap_equal_times_rules():
    """hb_snap_equal_times: equal within the measured spread -> equal;
    proportional otherwise; dead back-ends untouched."""
    assert hb.snap_equal_times([1.0, 1.02, 0.99], [0.05, 0.04, 0.03]) == [1.0033333333333332] * 3 or \
        len(set(hb.snap_equal_times([1.0, 1.02, 0.99], [0.05, 0.04, 0.03]))) == 1
    assert hb.snap_equal_times([1.0, 1.5], [0.05, 0.05]) == [1.0, 1.5]
    assert hb.snap_equal_times([1.0, 1.005], None, None, 0.01)[0] == hb.snap_equal_times([1.0, 1.005])[1]
    t = hb.snap_equal_times([1.0, 0.0, 1.01], [0.02, 0.0, 0.02], [True, False, True])
    assert t[1] == 0.0 and t[0] == t[2]
    assert hb.plan_allocation_n([1.0, 0.0, 1.0], 100) == [50, 0, 50]
