"""The drop-in check: the unmodified reference library (its own
calibrate / plan_allocation / run_hybrid / run_ea / cpu_executor) driving the
B200 backend through include/hbgpu/hetbench_gpu_executor.hpp
(oracle/ref_integration.cpp, built from /root/reference in the dev container
and shipped prebuilt)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_integration")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="reference integration binary not built")
def test_reference_library_drives_gpu_executor():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") >= 9
    assert "FAIL" not in r.stdout
