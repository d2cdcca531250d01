"""Per-phase Box kernel cost: time 16384 variants x S steps from states that
stay grounded, stay airborne, or follow the seeds (mixed), through
hb_run_states (wall clock; S large so the kernel dominates)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402


def main():
    n, steps = 16384, int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    only = sys.argv[1] if len(sys.argv) > 1 else None
    ex = hb.GpuExecutor(0)
    soa = hb.build_states(0, np.arange(n, dtype=np.uint64))
    base_p = soa[:3].T.reshape(n, 1, 3).copy()
    base_v = soa[3:6].T.reshape(n, 1, 3).copy()
    cases = {}
    p, v = base_p.copy(), base_v.copy()
    p[:, 0, 2] = 0.0
    v[:, 0, 2] = 0.0
    cases["grounded"] = (p, v)
    p, v = base_p.copy(), base_v.copy()
    p[:, 0, 2] = 1e5
    cases["airborne"] = (p, v)
    cases["seeds"] = (base_p, base_v)
    p, v = base_p.copy(), base_v.copy()
    p[0::2, 0, 2] = 0.0
    v[0::2, 0, 2] = 0.0
    p[1::2, 0, 2] = 1e5
    cases["mixed"] = (p, v)
    out = {}
    for name, (p, v) in cases.items():
        if only and name != only:
            continue
        ex.run_states(0, p, v, np.zeros((n, 0)), steps=100)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            ex.run_states(0, p, v, np.zeros((n, 0)), steps=steps)
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        out[name] = {"s": t, "ns_per_step": t / steps * 1e9, "cycles_per_step_at_1965": t / steps * 1.965e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
