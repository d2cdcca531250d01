"""Probe: humanoid blow-up states through run_states (fast vs generic kernel),
step counts around the failing step, each run timed (diagnostic)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2502_11129_b200 as hb  # noqa: E402

kind, N = 3, int(sys.argv[3]) if len(sys.argv) > 3 else 64
seeds = np.arange(N, dtype=np.uint64)
soa = hb.build_states(kind, seeds)
n = 32
pos = soa[: 3 * n].T.reshape(N, n, 3).copy()
vel = soa[3 * n: 6 * n].T.reshape(N, n, 3).copy()
rest = soa[6 * n:].T.copy()
pos[1::4, :, 0] += 999000.0
vel[1::4, :, 0] = 1000.0
which = sys.argv[1]
ex = hb.GpuExecutor(0, kernel=1 if which == "generic" else 0)
for steps in [int(x) for x in sys.argv[2].split(",")]:
    t = time.time()
    a = ex.run_states(kind, pos, vel, rest, steps=steps, seeds=seeds)
    print(which, steps, "fails", np.count_nonzero(a[1]), "first", a[1][a[1] > 0][:4], "%.3fs" % (time.time() - t),
          flush=True)
