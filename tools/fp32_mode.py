"""FP32 throughput mode (f3) vs the FP64 product path on B200: kernel rate of
both at the configs[2] size and the step-sweep size, the max relative
fitness error against FP64, and the EA parent-set agreement (run under
gpurun; JSON to stdout)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402
from paper_2502_11129_b200 import _lib  # noqa: E402

MODELS = ["box", "box_and_ball", "arm_with_rope", "humanoid", "cpg_hinge"]


def kernel_ms(ex, kind, n, steps, reps=3):
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


def main():
    ex64 = hb.GpuExecutor(0)
    ex32 = hb.GpuExecutor(0, precision=_lib.HB_PRECISION_FP32)
    out = {"models": {}}
    for m in MODELS:
        kind = hb.parse_model_kind(m)
        rows = []
        for n, steps in ((8192, 1000), (32768, 1000), (16384, 1000)):
            if m != "box" and n == 16384:
                continue
            t64 = kernel_ms(ex64, kind, n, steps)
            t32 = kernel_ms(ex32, kind, n, steps)
            seeds = np.arange(n, dtype=np.uint64)
            f64 = ex64.run(hb.BatchRequest(kind, seeds, steps)).results["fitness"]
            f32 = ex32.run(hb.BatchRequest(kind, seeds, steps)).results["fitness"]
            ae = np.abs(f32 - f64)
            err = ae / np.maximum(np.abs(f64), 1e-3)
            w = int(np.argmax(err))
            rows.append({"variants": n, "steps": steps, "fp64_ms": t64, "fp32_ms": t32,
                         "fp64_rate": n * steps / (t64 * 1e-3), "fp32_rate": n * steps / (t32 * 1e-3),
                         "speedup": t64 / t32, "max_rel_fitness_err": float(err.max()),
                         "mean_rel_fitness_err": float(err.mean()), "max_abs_fitness_err_m": float(ae.max()),
                         "worst_variant_fitness_m": float(f64[w]), "worst_variant_abs_err_m": float(ae[w]),
                         "frac_rel_err_above_1e-4": float(np.mean(err > 1e-4))})
            print(m, rows[-1], file=sys.stderr, flush=True)
        out["models"][m] = rows
    pop = 65536
    genomes = hb.rng_at(np.uint64(0x8F5D4C3B2A190807), np.arange(pop, dtype=np.uint64))
    agree = {}
    for m in ("box", "box_and_ball"):
        kind = hb.parse_model_kind(m)
        f64 = ex64.run(hb.BatchRequest(kind, genomes, 1000)).results["fitness"]
        f32 = ex32.run(hb.BatchRequest(kind, genomes, 1000)).results["fitness"]
        o64, o32 = np.argsort(-f64, kind="stable"), np.argsort(-f32, kind="stable")
        mu = pop // 2
        agree[m] = {"parent_set_overlap": len(set(o64[:mu].tolist()) & set(o32[:mu].tolist())) / mu,
                    "rank_identical_fraction": float(np.mean(o64[:mu] == o32[:mu]))}
    out["ea_selection_agreement_pop65536"] = agree
    print(json.dumps(out))


if __name__ == "__main__":
    main()
