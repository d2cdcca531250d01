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


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _bench_ranks(nproc, _label, *args):
    port = _free_port()  # the fixed numbers below are only labels
    env = dict(os.environ, HB_DIST_BACKEND="gloo")  # several ranks on one GPU: gloo, not NCCL
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", str(nproc), *args]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_two_ranks_batch_and_ea():
    """The multi-rank paths the driver's scaling run takes (torchrun, one
    rank per GPU; here two ranks share GPU 0 over gloo): calibrated shares,
    the max-over-ranks line, and the in-process N-context generation loop."""
    d = _bench_ranks(2, 29531, "--variants", "4096", "--sim-steps", "100", "--steps", "3", "--warmup", "3",
                     "--no-cpu-baseline")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    shares = d["config"]["splitter"]["shares"]
    assert sum(shares) == 8192 and len(shares) == 2
    st = _bench_ranks(2, 29533, "--variants", "8192", "--sim-steps", "100", "--steps", "3", "--warmup", "3",
                      "--no-cpu-baseline", "--scaling", "strong")
    assert st["scaling"] == "strong" and sum(st["config"]["splitter"]["shares"]) == 8192
    e = _bench_ranks(2, 29532, "--workload", "ea", "--population", "4096", "--generations", "2",
                     "--sim-steps", "100", "--steps", "3", "--warmup", "3")
    assert e["n_gpus"] == 2 and e["value"] > 0
    assert all(e["config"]["splitter"]["device_ok"])
