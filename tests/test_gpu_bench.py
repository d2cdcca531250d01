"""bench.py's JSON contract on small workloads (the driver parses these
lines): the default FP64 line, the FP32-mode line with its tolerance and
selection-agreement block, and the generation-loop line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"}


def _bench(*args):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_fp64_line():
    d = _bench("--variants", "2048", "--sim-steps", "50", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert KEYS <= set(d)
    assert d["dtype"] == "f64" and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["bound"] == "fp64" and 0 < d["roofline"]["frac"] <= 1.0
    assert d["roofline"]["kernel"] == "box_kernel"
    assert "fp32" not in d


def test_bench_fp32_mode_line():
    d = _bench("--model", "box_and_ball", "--variants", "4096", "--sim-steps", "200", "--steps", "3",
               "--warmup", "3", "--no-cpu-baseline", "--precision", "fp32")
    assert KEYS <= set(d)
    assert d["dtype"].startswith("f32") and d["roofline"]["bound"] == "fp32"
    assert "[FP32 mode]" in d["config"]["workload"]
    f = d["fp32"]
    assert f["max_rel_fitness_err"] <= 1e-4  # box_and_ball's stated tolerance (test_gpu_fp32.py)
    assert f["parent_set_overlap"] >= 0.99


def test_bench_ea_line():
    d = _bench("--workload", "ea", "--population", "4096", "--generations", "2", "--sim-steps", "100",
               "--steps", "3", "--warmup", "3")
    assert KEYS - {"roofline"} <= set(d)  # the loop line reports phases, not a kernel roofline
    assert d["value"] > 0 and d["host_overhead_us_per_generation"] >= 0
