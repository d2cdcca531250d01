"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): each model through hb_run_batch (device
initialisers), the generation loop for Box (queued, cluster sort) and
BoxAndBall (checked), the device-wide sort path, the FP32 throughput
mode, the generic kernel variant and the Box zero-copy call."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402
from paper_2502_11129_b200 import _lib  # noqa: E402


def main():
    ex = hb.GpuExecutor(0)
    rng = np.random.default_rng(1)
    for kind in range(5):
        seeds = rng.integers(0, 2**63, 1000, dtype=np.uint64)
        ex.run(hb.BatchRequest(kind, seeds, 20))
    # the saturated-regime shapes (register-capped multibody kernels, U = 1 / 2)
    for kind, n in ((1, 65536), (2, 65536), (4, 65536)):
        ex.run(hb.BatchRequest(kind, np.arange(n, dtype=np.uint64), 2))
    ex.reserve(3, 4096)
    hb.run_ea(0, 4096, 2, 20, ex, seed=1)
    hb.run_ea(0, 70000, 1, 5, ex, seed=1)
    hb.run_ea(1, 2048, 2, 10, ex, seed=1)
    fp32 = hb.GpuExecutor(0, precision=_lib.HB_PRECISION_FP32)
    gen = hb.GpuExecutor(0, kernel=_lib.HB_KERNEL_GENERIC)
    for kind in range(5):
        seeds = rng.integers(0, 2**63, 700, dtype=np.uint64)
        fp32.run(hb.BatchRequest(kind, seeds, 15))
        gen.run(hb.BatchRequest(kind, seeds, 15))
    s = _lib.pinned.empty(3000, np.uint64)
    s[:] = rng.integers(0, 2**63, 3000, dtype=np.uint64)
    out = _lib.pinned.empty(3000, _lib.RESULT_DTYPE)
    wall = C.c_double(0)
    assert _lib.lib.hb_run_batch(ex.ctx.handle, 0, _lib.ptr(s), 3000, 100, _lib.ptr(out), None,
                                 C.byref(wall)) == _lib.HB_OK
    print("sanitize probe: ok")


if __name__ == "__main__":
    main()
