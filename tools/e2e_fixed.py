"""Fixed (step-count independent) cost of the zero-copy drop-in call, by
layer: GpuExecutor.run (Python mirror), run_raw, and the bare C-ABI call
hb_run_batch through ctypes, with pinned seeds/results, at 1 / 16 / 1000
steps (wall clock, median of 200)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402
from paper_2502_11129_b200 import _lib  # noqa: E402


def med(fn, reps=200):
    for _ in range(20):
        fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    t = np.array(t) * 1e6
    return np.median(t), t.min()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    only_abi = len(sys.argv) > 2
    ex = hb.GpuExecutor(0)
    seeds = _lib.pinned.empty(n, np.uint64)
    seeds[:] = np.arange(n, dtype=np.uint64)
    out = _lib.pinned.empty(n, hb.RESULT_DTYPE)
    lib = _lib.lib
    h = ex.ctx.handle
    sp, op = _lib.ptr(seeds), _lib.ptr(out)
    wall = C.c_double(0)
    for steps in (1, 16, 1000):
        req = hb.BatchRequest(0, seeds, steps)
        rows = []
        if not only_abi:
            rows.append(("run", med(lambda: ex.run(req))))
            rows.append(("run_raw", med(lambda: ex.run_raw(0, seeds, steps))))
        rows.append(("hb_run_batch", med(lambda: lib.hb_run_batch(h, 0, sp, n, steps, op, None, C.byref(wall)))))
        print(f"steps {steps:5d}: " + "  ".join(f"{k} {m:6.1f} (min {mn:6.1f}) us" for k, (m, mn) in rows))


if __name__ == "__main__":
    main()
