"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): each model through hb_run_batch (device
initialisers), the generation loop for Box (queued, cluster sort) and
BoxAndBall (checked), and the device-wide sort path."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402


def main():
    ex = hb.GpuExecutor(0)
    rng = np.random.default_rng(1)
    for kind in range(5):
        seeds = rng.integers(0, 2**63, 1000, dtype=np.uint64)
        ex.run(hb.BatchRequest(kind, seeds, 20))
    hb.run_ea(0, 4096, 2, 20, ex, seed=1)
    hb.run_ea(0, 70000, 1, 5, ex, seed=1)
    hb.run_ea(1, 2048, 2, 10, ex, seed=1)
    print("sanitize probe: ok")


if __name__ == "__main__":
    main()
