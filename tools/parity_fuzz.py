"""Parity fuzz across the dispatcher's shape boundaries (run under gpurun).

For every model, batch sizes around each kernel-selection threshold (CTA
edges, the two-lane CpgHinge limit 12 288, the register-capped shapes from
65 536) and several step counts, random 64-bit seeds:
  * the optimised kernels against the reference-order generic kernel, every
    record of the batch, bit for bit;
  * a strided subsample against the oracle restatement (oracle/hb_oracle.c)
    and, for the reference's own models, against the reference library
    compiled in place (oracle/_ref) — test infrastructure, not product.
One line per case; a summary line at the end; exit code = failures.

    python tools/parity_fuzz.py [--quick] > profiles/r02_parity_fuzz.txt
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2502_11129_b200 as hb  # noqa: E402
from paper_2502_11129_b200 import _lib  # noqa: E402

SIZES = [1, 31, 33, 1000, 12288, 12289, 16385, 65535, 65536, 131072]
STEPS = [1, 7, 300, 2000]
MODELS = ["box", "box_and_ball", "arm_with_rope", "humanoid", "cpg_hinge"]


def main():
    quick = "--quick" in sys.argv
    sizes = SIZES[:6] if quick else SIZES
    fast = hb.GpuExecutor(0)
    gen = hb.GpuExecutor(0, kernel=_lib.HB_KERNEL_GENERIC)
    rng = np.random.default_rng(20261017)
    fails = cases = records = 0
    t0 = time.time()
    for kind, name in enumerate(MODELS):
        for n in sizes:
            for steps in STEPS:
                seeds = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
                a = fast.run(hb.BatchRequest(kind, seeds, steps)).results
                b = gen.run(hb.BatchRequest(kind, seeds, steps)).results
                ok_gen = np.array_equal(a, b)
                idx = np.unique(np.concatenate([np.arange(0, n, max(1, n // 64)), [n - 1]]))
                ok_orc = np.array_equal(a[idx], O.simulate_batch(kind, seeds[idx], steps).results)
                ok_ref = True
                if kind < 4 and O.ref_available():
                    rc, want, _, _, msg = O.ref_cpu_run(kind, seeds[idx], steps, 0)
                    ok_ref = rc == 0 and np.array_equal(a[idx], want)
                ok = ok_gen and ok_orc and ok_ref
                cases += 1
                records += n
                fails += 0 if ok else 1
                print(f"{'PASS' if ok else 'FAIL'} {name:13s} n={n:6d} steps={steps:4d} "
                      f"kernel={hb.kernel_name(kind, n)} generic={ok_gen} oracle({len(idx)})={ok_orc} "
                      f"reference={ok_ref if kind < 4 else 'n/a'}", flush=True)
    print(f"summary: {cases} cases, {records} records vs the generic kernel, {fails} failures, "
          f"{time.time() - t0:.1f} s", flush=True)
    fast.ctx.close()
    gen.ctx.close()
    return fails


if __name__ == "__main__":
    sys.exit(main())
