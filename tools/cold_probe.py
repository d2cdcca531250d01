"""Cold-start cost of the drop-in call: a fresh context's first hb_run_batch
per model (buffer growth, lazy kernel load, NVML init with the monitor on)
against the warm second call, at the paper's calibrate probe sizes.
Run with HB_TRACE=1 for the host phase split."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402

monitor = len(sys.argv) > 1 and sys.argv[1] == "monitor"
for kind, n in ((0, 512000), (1, 512000), (2, 256000), (3, 32768), (4, 32768)):
    t0 = time.perf_counter()
    ex = hb.GpuExecutor(0, monitor=monitor)
    t1 = time.perf_counter()
    seeds = np.arange(n, dtype=np.uint64)
    walls = []
    for _ in range(3):
        r = ex.run(hb.BatchRequest(kind, seeds, 100))
        walls.append(r.wall_time_s)
    print(f"kind {kind} n {n}: ctx create {1e3 * (t1 - t0):.1f} ms, calls (wall_time_s) "
          + " ".join(f"{1e3 * w:.2f}" for w in walls) + " ms", flush=True)
    ex.ctx.close()
