"""Generate tests/golden/golden.json from the REFERENCE itself.

Runs in the dev container only (needs oracle/_ref/libhetbench_ref.so, i.e. the
unmodified /root/reference/proj/src compiled by oracle/Makefile).  The output
is committed; the GPU box never reads /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402


def hx(x: int) -> str:
    return "%016x" % x


def fbits(x: float) -> str:
    return hx(int(np.float64(x).view(np.uint64)))


def main():
    O.build(with_ref=True)
    assert O.ref_available(), "reference library not built"
    g = {"source": "oracle/_ref/libhetbench_ref.so (reference proj/src compiled in place)",
         "dt": O.DT}

    # 1. simulate(kind, seed, steps) for a grid (Appendix A of SURVEY.md is a subset).
    sim = []
    for kind in range(4):
        for seed in (0, 1, 2, 3, 7, 42, 1234567, 2**63 + 5, 2**64 - 1):
            for steps in (1, 2, 10, 100, 1000):
                rc, r, msg = O.ref_simulate(kind, seed, steps)
                assert rc == 0, msg
                sim.append({"kind": kind, "seed": str(seed), "steps": steps,
                            "fitness_bits": fbits(r[1]), "checksum": hx(r[2])})
    g["simulate"] = sim

    # 2. Acceptance C1 recipe (acceptance.cpp:200-218): 200 (model, steps)
    #    cells with seeds rng::at(0xACC1, i).
    c1 = []
    for i in range(200):
        kind = i % 4
        steps = (10, 100, 1000)[(i // 4) % 3]
        seed = O.ref().hbref_rng_at(0xACC1, i)
        rc, r, msg = O.ref_simulate(kind, seed, steps)
        assert rc == 0
        c1.append({"i": i, "kind": kind, "steps": steps, "seed": str(seed),
                   "fitness_bits": fbits(r[1]), "checksum": hx(r[2])})
    g["c1"] = c1

    # 3. build_model initial states (bits) for a few seeds per model.
    bm = []
    import ctypes as C
    for kind in range(4):
        for seed in (0, 5, 42, 2**64 - 1):
            n, m = O.BODIES[kind], O.CONSTRAINTS[kind]
            pos = np.zeros(3 * n); vel = np.zeros(3 * n); rest = np.zeros(max(m, 1))
            O.ref().hbref_build_model(kind, seed, O._dp(pos), O._dp(vel), O._dp(rest), None, None,
                                      None)
            bm.append({"kind": kind, "seed": str(seed),
                       "pos_bits": [fbits(x) for x in pos], "vel_bits": [fbits(x) for x in vel],
                       "rest_bits": [fbits(x) for x in rest[:m]]})
    g["build_model"] = bm

    # 4. Known answers on explicit states (test_simkernel.cpp:106-126,182-186).
    ka = {}
    buf = C.create_string_buffer(512)

    def ref_step(kind, pos, vel, dt, seed):
        pos = np.ascontiguousarray(pos, dtype=np.float64).ravel().copy()
        vel = np.ascontiguousarray(vel, dtype=np.float64).ravel().copy()
        rc = O.ref().hbref_step_state(kind, O._dp(pos), O._dp(vel), dt, seed, buf, 512)
        return rc, pos, vel, buf.value.decode()

    rc, p, v, _ = ref_step(0, [0.3, -0.2, 0.0], [0, 0, 0], O.DT, 0)
    ka["rest_on_ground"] = {"rc": rc, "pos_bits": [fbits(x) for x in p],
                            "vel_bits": [fbits(x) for x in v]}
    rc, p, v, _ = ref_step(0, [0.0, 0.0, 5.0], [0, 0, 0], O.DT, 5)
    ka["free_fall"] = {"rc": rc, "pos_bits": [fbits(x) for x in p],
                       "vel_bits": [fbits(x) for x in v]}
    p0, v0, _ = O.build_model(0, 0)
    rc, p, v, msg = ref_step(0, p0, [0.0, 0.0, 1e9], O.DT, 0)
    ka["blowup_vz_1e9"] = {"rc": rc, "message": msg}
    g["known_answers"] = ka

    # 5. Intermediate trajectories (full state bits) for trajectory parity.
    tr = []
    for kind in range(4):
        n = O.BODIES[kind]
        for steps in (1, 7, 64, 500):
            pos = np.zeros(3 * n); vel = np.zeros(3 * n); t = C.c_double(0)
            rc = O.ref().hbref_trajectory(kind, 11, steps, O._dp(pos), O._dp(vel), C.byref(t))
            tr.append({"kind": kind, "seed": "11", "steps": steps, "rc": rc,
                       "pos_bits": [fbits(x) for x in pos], "vel_bits": [fbits(x) for x in vel],
                       "time_bits": fbits(t.value)})
    g["trajectory"] = tr

    # 6. Splitter: acceptance C3 recipe (acceptance.cpp:273-305) + reference splits.
    plans = []
    for i in range(1000):
        key = 0xACC3
        base = i * 8
        t_cpu = 1e-6 + (10.0 - 1e-6) * ((O.ref().hbref_rng_at(key, base) >> 11) * 2.0**-53)
        t_acc = 1e-6 + (10.0 - 1e-6) * ((O.ref().hbref_rng_at(key, base + 1) >> 11) * 2.0**-53)
        n = 1 + O.ref().hbref_rng_at(key, base + 2) % 10000
        p = O.ref_plan_allocation(t_cpu, t_acc, n)
        plans.append({"t_cpu_bits": fbits(t_cpu), "t_accel_bits": fbits(t_acc), "n": n,
                      "n_cpu": p[1], "n_accel": p[2], "frac_bits": fbits(p[4])})
    g["plan_allocation"] = plans
    ref_splits = []
    for (tc, ta, n, cok, aok) in ((2.0, 2.0, 100, 1, 1), (2.0, 6.0, 100, 1, 1),
                                  (1.0, 1e9, 10, 1, 1), (19.0, 1.0, 10, 1, 1),
                                  (1.0, 1e-9, 10, 1, 1), (2.0, 0.0, 10, 0, 1),
                                  (2.0, 0.0, 10, 1, 0)):
        p = O.ref_plan_allocation(tc, ta, n, bool(cok), bool(aok))
        ref_splits.append({"t_cpu": tc, "t_accel": ta, "n": n, "cpu_ok": cok, "accel_ok": aok,
                           "n_cpu": p[1], "n_accel": p[2], "frac_bits": fbits(p[4])})
    g["plan_reference_splits"] = ref_splits

    # 7. run_ea trajectories (ea.cpp:33-105) over the reference cpu_executor.
    eas = []
    for (kind, pop, gens, steps, seed) in ((0, 8, 3, 40, 7), (1, 16, 4, 60, 42),
                                           (2, 8, 2, 30, 0), (3, 8, 2, 20, 3),
                                           (1, 256, 3, 100, 0)):
        gen, fit = O.ref_run_ea(kind, pop, gens, steps, seed, workers=2)
        eas.append({"kind": kind, "pop": pop, "generations": gens, "steps": steps, "seed": seed,
                    "genomes": [hx(int(x)) for x in gen], "fitness_bits": [fbits(x) for x in fit]})
    g["run_ea"] = eas

    # 8. Reference blow-up text (simkernel.cpp:165-169) after s normal steps
    #    and one step with body 0 kicked to v.z = 1e9: fail_step = s + 1.
    msgs = []
    for s_before in (0, 9, 999, 4999):
        rc = O.ref().hbref_blowup_after(0, 3, s_before, buf, 512)
        assert rc == 1
        msgs.append({"fail_step": s_before + 1, "message": buf.value.decode()})
    g["blowup_messages"] = msgs

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print("wrote", path, os.path.getsize(path), "bytes")

    # CpgHinge (kind 4) is NOT in the reference: its values come from the
    # oracle that defines it (oracle/hb_oracle.c) — a regression anchor only.
    cg = {"source": "oracle/_build/libhboracle.so (model defined there; parity unpinned)",
          "simulate": []}
    for seed in (0, 1, 42, 2**64 - 1):
        for steps in (1, 10, 1000, 5000):
            rc, r, _ = O.simulate(4, seed, steps)
            assert rc == 0
            cg["simulate"].append({"seed": str(seed), "steps": steps, "fitness_bits": fbits(r[1]),
                                   "checksum": hx(r[2])})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpg_golden.json")
    with open(path, "w") as f:
        json.dump(cg, f, indent=0, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
