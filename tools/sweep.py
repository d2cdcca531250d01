"""The paper's sweeps on B200 (run under gpurun):

  * variant sweep — paper grid 32..512 000 per model, 1 000 steps
    (proj/configs/full_grid.toml:27-38), e2e wall of the drop-in call
    (3 repetitions, Student-t CI95 like monitor.cpp:76-105) and the
    saturation knee found by the reference's own detect_saturation_knee
    (monitor.cpp:184-203, via oracle/_ref) on the measured curve;
  * step sweep (BASELINE config 4) — 100..20 000 steps at 32 768 variants
    for all four models, kernel-only and e2e rates;
  * reference CPU rate per model on the host cores (bounded sample).

    python tools/sweep.py --out profiles/r02_sweeps.json [--quick]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_11129_b200 as hb  # noqa: E402

GRID = {
    "box": [32, 128, 256, 512, 1024, 2056, 4096, 8192, 16384, 32768, 65536, 131072, 256000, 512000],
    "box_and_ball": [32, 128, 256, 512, 1024, 2056, 4096, 8192, 16384, 32768, 65536, 131072, 256000,
                     512000],
    "arm_with_rope": [32, 128, 256, 512, 1024, 2056, 4096, 8192, 16384, 32768, 65536, 131072, 256000],
    "humanoid": [32, 128, 256, 512, 1024, 2056, 4096, 8192, 16384, 32768],
    "cpg_hinge": [32, 128, 256, 512, 1024, 2056, 4096, 8192, 16384, 32768, 65536, 131072],
}
STEPS = [100, 200, 500, 1000, 2000, 5000, 10000, 20000]
W_ALG = {"box": 16, "box_and_ball": 200, "arm_with_rope": 2040, "humanoid": 8240, "cpg_hinge": 2204}


def t_ci95(samples):
    st = hb.summarize(samples)
    return st.mean, st.ci95_low, st.ci95_high


def e2e_walls(ex, kind, n, steps, reps):
    from paper_2502_11129_b200 import _lib
    seeds = _lib.pinned.empty(n, np.uint64)
    seeds[:] = np.arange(n, dtype=np.uint64)
    req = hb.BatchRequest(kind, seeds, steps)
    ex.run(req)  # warm-up (allocations)
    walls = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ex.run(req)
        walls.append(time.perf_counter() - t0)
    return walls


def kernel_ms(ex, kind, n, steps, reps=3):
    import torch
    ctx = ex.ctx
    ctx.stage(kind, np.arange(n, dtype=np.uint64))
    ext = torch.cuda.ExternalStream(ctx.stream)
    ctx.launch(steps)
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        ctx.launch(steps)
        e1.record(ext)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def knee(ns, walls):
    n, regime = hb.detect_saturation_knee(list(zip(ns, walls)))
    return {"n": int(n), "regime": regime.name}


def cpu_rate(kind, steps=1000):
    import oracle as O
    if int(kind) == 4:  # CpgHinge: no reference model; the oracle port, all host threads
        cores = os.cpu_count() or 1
        n = max(64 * cores, 4096)
        steps = max(10, min(steps, int(3.0 * cores / (n * 1300e-9))))
        seeds = np.arange(n, dtype=np.uint64)
        t0 = time.perf_counter()
        O.simulate_batch(4, seeds, steps, threads=cores)
        wall = time.perf_counter() - t0
        return {"value": n * steps / wall, "cores": cores, "kind": "port",
                "sample": f"{n} variants x {steps} steps"}
    if not O.ref_available():
        return None
    cores = O.ref_hardware_concurrency()
    per_ns = {0: 58, 1: 298, 2: 2110, 3: 8190}[int(kind)]
    n = max(64 * cores, 4096)
    steps = max(10, min(steps, int(3.0 * cores / (n * per_ns * 1e-9))))
    seeds = np.arange(n, dtype=np.uint64)
    best = None
    for _ in range(2):
        rc, _, wall, _, _ = O.ref_cpu_run(int(kind), seeds, steps, workers=0)
        best = wall if best is None else min(best, wall)
    return {"value": n * steps / best, "cores": cores, "sample": f"{n} variants x {steps} steps"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweeps.json")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--models", default="box,box_and_ball,arm_with_rope,humanoid,cpg_hinge")
    a = ap.parse_args()
    ex = hb.GpuExecutor(0)
    peak, _ = ex.ctx.fp64_peak()
    res = {"fp64_peak_ops": peak, "variant_sweep": {}, "step_sweep": {}, "cpu_reference": {}}
    models = a.models.split(",")
    for m in models:
        kind = hb.parse_model_kind(m)
        res["cpu_reference"][m] = cpu_rate(kind)
        rows = []
        for n in (GRID[m][::3] if a.quick else GRID[m]):
            walls = e2e_walls(ex, kind, n, 1000, 3)
            mean, lo, hi = t_ci95(walls)
            rows.append({"n": n, "wall_mean_s": mean, "ci95": [lo, hi], "walls": walls,
                         "rate_vs_per_s": n * 1000 / mean})
            print(m, "n", n, "wall %.6f" % mean, flush=True)
        res["variant_sweep"][m] = {"steps": 1000, "rows": rows,
                                   "knee": knee([r["n"] for r in rows], [r["wall_mean_s"] for r in rows])}
        srows = []
        for s in (STEPS[::2] if a.quick else STEPS):
            ops0 = ex.ctx.work_counter()
            km = kernel_ms(ex, kind, 32768, s)
            ops = (ex.ctx.work_counter() - ops0) / 4  # kernel_ms launches 1 warm-up + 3 timed
            walls = e2e_walls(ex, kind, 32768, s, 2)
            rate = 32768 * s / (km * 1e-3)
            srows.append({"steps": s, "kernel_ms": km, "rate_kernel": rate,
                          "rate_e2e": 32768 * s / float(np.min(walls)),
                          # Box: executed ops (z elided exactly when grounded), W_alg beside
                          "roofline_frac": (ops / (km * 1e-3) / peak if m == "box" else
                                            W_ALG[m] * rate / peak),
                          "roofline_frac_w_alg": W_ALG[m] * rate / peak})
            print(m, "steps", s, "kernel %.3f ms" % km, flush=True)
        res["step_sweep"][m] = {"variants": 32768, "rows": srows}
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
