"""Where the end-to-end time of the drop-in call goes (run under gpurun).

    python tools/e2e_breakdown.py [--model box] [--variants 16384] [--sim-steps 1000]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_11129_b200 as hb  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(t)), 1e6 * float(np.min(t))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="box")
    ap.add_argument("--variants", type=int, default=16384)
    ap.add_argument("--sim-steps", type=int, default=1000)
    a = ap.parse_args()
    kind = hb.parse_model_kind(a.model)
    seeds = np.arange(a.variants, dtype=np.uint64)
    ex = hb.GpuExecutor(0)
    ctx = ex.ctx
    req = hb.BatchRequest(kind, seeds, a.sim_steps)
    rows = []
    rows.append(("GpuExecutor.run (drop-in, Python)", timeit(lambda: ex.run(req))))
    rows.append(("run_raw (ctypes hb_run_batch)", timeit(lambda: ex.run_raw(kind, seeds, a.sim_steps))))
    rows.append(("hb_stage (host init/copy + H2D + sync)", timeit(lambda: ctx.stage(kind, seeds))))

    def launch_sync():
        ctx.launch(a.sim_steps)
        ctx.synchronize()
    rows.append(("hb_launch + sync (kernel)", timeit(launch_sync)))
    rows.append(("hb_launch + sync, 1 step", timeit(lambda: (ctx.launch(1), ctx.synchronize()))))
    rows.append(("hb_fetch (D2H + assemble)", timeit(ctx.fetch)))
    for name, (med, mn) in rows:
        print(f"{name:45s} median {med:9.1f} us   min {mn:9.1f} us")


if __name__ == "__main__":
    main()
