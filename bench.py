#!/usr/bin/env python
"""bench.py — variant-steps/sec of the B200 batched-simulation hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model box] [--variants 16384] [--sim-steps 1000]

A bench "step" is one pass of the hot path over one batch: every variant of
the per-GPU batch simulated through all `--sim-steps` physics steps (one
persistent-kernel launch).  Default workload = BASELINE.json configs[1]:
box, 16 384 variants x 1 000 steps per GPU (weak scaling for N > 1: each rank
gets a contiguous 16 384-seed slice of the global batch from the N-way
splitter).

value : device-resident inputs, CUDA events on the kernel's stream around
        each launch, L2 flushed (256 MiB write) between launches outside the
        event pair; max over ranks.
e2e   : the drop-in call GpuExecutor.run -> hb_run_batch with HOST seeds:
        host initialiser, H2D of the initial state, kernel, D2H of the
        32-byte results, all inside the timed region (wall clock, max over ranks).
--impl reference : the reference's own cpu_executor (oracle/_ref, compiled
        from /root/reference/proj/src) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "variant-steps/sec (whole box) vs #variants & steps; speedup over host-CPU ref"
MODELS = ("box", "box_and_ball", "arm_with_rope", "humanoid", "cpg_hinge")
# Algorithmic FP64 ops per variant-step (add/sub/mul/div/sqrt = 1,
# compares excluded): 16n + 8m*(19 + sqrt + div).
# cpg_hinge (not in the reference): 16*9 + 8*12*21 + 4 joints x 11 CPG/actuation ops.
W_ALG = {"box": 16, "box_and_ball": 200, "arm_with_rope": 2040, "humanoid": 8240, "cpg_hinge": 2204}
BODIES = {"box": 1, "box_and_ball": 2, "arm_with_rope": 12, "humanoid": 32, "cpg_hinge": 9}
CONS = {"box": 0, "box_and_ball": 1, "arm_with_rope": 11, "humanoid": 46, "cpg_hinge": 12}
EXTRA_ROWS = {"cpg_hinge": 16}
PER_VS_CORE_NS = {0: 58, 1: 298, 2: 2110, 3: 8190, 4: 1700}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="box", choices=MODELS)
    ap.add_argument("--variants", type=int, default=16384,
                    help="variants per GPU (weak scaling) or in total (--scaling strong)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: --variants per GPU (the default line); strong: --variants in total, "
                         "split over the GPUs by the splitter (BASELINE configs[3]: 32768 variants at "
                         "1/2/4/8 GPUs)")
    ap.add_argument("--sim-steps", type=int, default=1000)
    ap.add_argument("--workload", default="batch", choices=["batch", "ea"],
                    help="batch = one simulate() pass per step (configs[1]); ea = full generation "
                         "loop per step (configs[4]: evaluate, fitness gather, select)")
    ap.add_argument("--population", type=int, default=65536, help="ea: population size (global)")
    ap.add_argument("--generations", type=int, default=5, help="ea: generations per step")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="fp64 = the bit-exact product path; fp32 = the opt-in FP32 throughput mode "
                         "(multi-body models; SURVEY §8 f3): the line adds its fitness error and EA "
                         "selection agreement against the FP64 product on the same seeds")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload_name(a):
    strong = getattr(a, "scaling", "weak") == "strong"
    tag = ""
    if (a.model, a.variants, a.sim_steps) == ("box", 16384, 1000) and not strong:
        tag = " (BASELINE configs[1])"
    elif a.variants == 32768 and strong:
        tag = " (BASELINE configs[3] point)"
    mode = " [FP32 mode]" if getattr(a, "precision", "fp64") == "fp32" and a.model != "box" else ""
    per = "in total, split over the GPUs" if strong else "per GPU"
    return f"{a.model} {a.variants} variants x {a.sim_steps} steps {per}{tag}{mode}"


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_traffic(model, variants, sim_steps):
    """dram bytes per launch from the committed ncu capture, if one matches."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{model}/{variants}/{sim_steps}")
    except (OSError, ValueError):
        return None


def host_cpu():
    """lscpu topology of the host the CPU baseline ran on (BASELINE.md §3:
    state the core count and sockets, not only hardware_concurrency)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
    except (OSError, subprocess.SubprocessError):
        return info
    keys = {"Model name": "model", "Socket(s)": "sockets", "Core(s) per socket": "cores_per_socket",
            "Thread(s) per core": "threads_per_core", "CPU(s)": "logical_cpus"}
    for line in out.splitlines():
        k, _, v = line.partition(":")
        k = k.strip()
        if k in keys:
            v = v.strip()
            info[keys[k]] = int(v) if v.isdigit() else v
    if isinstance(info.get("sockets"), int) and isinstance(info.get("cores_per_socket"), int):
        info["physical_cores"] = info["sockets"] * info["cores_per_socket"]
    return info


CPU_SAMPLE_S = 25.0  # CPU-work budget of the in-run baseline sample (estimate; ~10 s measured)


def cpu_reference_rate(model_idx, n, sim_steps):
    """Reference cpu_executor(workers = hardware_concurrency) on the host, on a
    bounded sample of the workload (the full batch when one run is cheap,
    else N' = max(64 x cores, 4096) variants), repeated for ~CPU_SAMPLE_S of
    CPU work; reports the best run (the most favourable CPU figure) and the
    median."""
    import oracle as O
    if model_idx == 4:
        return cpu_port_rate(model_idx, n, sim_steps)
    if not O.ref_available():
        return None
    cores = O.ref_hardware_concurrency()
    per_run_s = n * sim_steps * PER_VS_CORE_NS[model_idx] * 1e-9 / cores
    n_s = n if per_run_s <= 10.0 else min(n, max(64 * cores, 4096))
    per_run_s *= n_s / n
    reps = int(min(400, max(3, CPU_SAMPLE_S / max(per_run_s, 1e-6))))
    seeds = np.arange(n_s, dtype=np.uint64)
    walls = []
    for _ in range(reps):
        rc, out, wall, _, msg = O.ref_cpu_run(model_idx, seeds, sim_steps, workers=0)
        if rc != 0:
            raise RuntimeError("reference cpu_executor failed: " + msg)
        walls.append(wall)
    best = min(walls)
    return {"value": n_s * sim_steps / best, "unit": "variant-steps/s", "cores": cores,
            "kind": "reference", "host": host_cpu(),
            "median_value": n_s * sim_steps / float(np.median(walls)),
            "sample": f"{MODELS[model_idx]} {n_s} variants x {sim_steps} steps, seeds 0..{n_s - 1}, "
                      f"reference cpu_executor(workers=0 -> {cores} threads), best of {reps} runs "
                      f"({sum(walls):.1f} s)",
            "walls_s_min_max": [best, max(walls)]}


def cpu_port_rate(model_idx, n, sim_steps, reps=3):
    """CpgHinge has no reference implementation: time its defining C oracle
    (oracle/hb_oracle.c, one pthread per host core) instead — kind "port"."""
    import oracle as O
    cores = os.cpu_count() or 1
    est_s = n * sim_steps * PER_VS_CORE_NS[model_idx] * 1e-9 / cores * reps
    n_s = n if est_s <= CPU_SAMPLE_S else min(n, max(64 * cores, 4096))
    seeds = np.arange(n_s, dtype=np.uint64)
    walls = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.simulate_batch(model_idx, seeds, sim_steps, cores)
        walls.append(time.perf_counter() - t0)
    return {"value": n_s * sim_steps / min(walls), "unit": "variant-steps/s", "cores": cores,
            "kind": "port", "host": host_cpu(),
            "sample": f"{MODELS[model_idx]} {n_s} variants x {sim_steps} steps through the model's "
                      f"defining C oracle ({cores} threads; the reference has no such model), best of {reps}",
            "walls_s": walls}


# ---------------------------------------------------------------- reference arm
def run_reference(a, ws, rank):
    if rank != 0:
        return
    import oracle as O
    k = MODELS.index(a.model)
    base = {"metric": METRIC, "impl": "reference", "unit": "variant-steps/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "higher_is_better": True, "dtype": "f64",
            "data": "synthetic (seeds 0..N-1, build_model initial states)",
            "config": {"workload": workload_name(a), "model": a.model,
                       "variants_per_gpu": a.variants, "sim_steps": a.sim_steps}}
    if k == 4:
        print(json.dumps({"impl": "reference",
                          "unavailable": "cpg_hinge is not a reference model (SPEC.md:101); "
                                         "its cpu_baseline is the defining oracle port"}))
        return
    if not O.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libhetbench_ref.so was not built"}))
        return
    cores = O.ref_hardware_concurrency()
    if a.workload == "ea":
        # the reference's own run_ea over cpu_executor(workers = all threads)
        per_vs_core_ns = PER_VS_CORE_NS[k]
        G = a.generations
        pop = a.population
        budget = 10.0 * cores / (per_vs_core_ns * 1e-9) / a.sim_steps  # variants per step
        while pop > 64 * cores and (pop + G * pop // 2) > budget:
            pop //= 2
        evaluated = pop + G * (pop // 2)
        for _ in range(a.warmup):
            O.ref_run_ea(k, pop, G, a.sim_steps, 0, workers=0)
        t0 = time.perf_counter()
        for _ in range(a.steps):
            O.ref_run_ea(k, pop, G, a.sim_steps, 0, workers=0)
        total = time.perf_counter() - t0
        value = evaluated * a.sim_steps * a.steps / total
        sample = (f"reference run_ea {a.model} pop {pop} (of {a.population}) x {G} generations x "
                  f"{a.sim_steps} steps over cpu_executor(workers=0 -> {cores} threads)")
        base["config"].update({"workload": f"ea: run_ea {a.model} pop {a.population} x {G} "
                                           f"generations x {a.sim_steps} steps (BASELINE configs[4])"})
        base.update({"value": value, "ms_per_step": 1e3 * total / a.steps,
                     "cpu_baseline": {"value": value, "unit": "variant-steps/s", "cores": cores,
                                      "kind": "reference", "sample": sample, "host": host_cpu()},
                     "e2e": {"value": value, "unit": "variant-steps/s", "h2d_bytes_per_step": 0,
                             "d2h_bytes_per_step": 0},
                     "vs_baseline": None, "scaling": "strong"})
        print(json.dumps(base))
        return
    n_total = a.variants * a.gpus if a.scaling == "weak" else a.variants
    # bounded per-step sample: ~10 s of host time per step at most
    per_vs_core_ns = PER_VS_CORE_NS[k]
    max_vs = 10.0 * cores / (per_vs_core_ns * 1e-9)
    n_s = n_total if n_total * a.sim_steps <= max_vs else max(64 * cores, int(max_vs // a.sim_steps))
    n_s = min(n_s, n_total)
    seeds = np.arange(n_s, dtype=np.uint64)
    for _ in range(a.warmup):
        O.ref_cpu_run(k, seeds, a.sim_steps, workers=0)
    t0 = time.perf_counter()
    walls = []
    for _ in range(a.steps):
        rc, _, wall, _, msg = O.ref_cpu_run(k, seeds, a.sim_steps, workers=0)
        if rc != 0:
            raise RuntimeError(msg)
        walls.append(wall)
    total = time.perf_counter() - t0
    value = n_s * a.sim_steps * a.steps / total
    sample = (f"{a.model} {n_s} of {n_total} variants x {a.sim_steps} steps per bench step, "
              f"reference cpu_executor(workers=0 -> {cores} threads)")
    base.update({"value": value, "ms_per_step": 1e3 * total / a.steps,
                 "cpu_baseline": {"value": value, "unit": "variant-steps/s", "cores": cores,
                                  "kind": "reference", "sample": sample, "host": host_cpu()},
                 "e2e": {"value": value, "unit": "variant-steps/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0},
                 "vs_baseline": None, "scaling": "weak"})
    print(json.dumps(base))


def latency_bound(a, n, ops_exec, kernel_ms, clk):
    """Dependent-chain latency roofline of the Box kernel and
    of the CpgHinge kernel (64 serial projections per step)."""
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    if a.model == "cpg_hinge":
        # 8 sweeps x 8 serial slots (every link of the core body is serial),
        # each projection a ~166-cycle dependent chain: 3 DADD (d), 3 DMUL +
        # 2 DADD (d^2), MUFU + 7 FP64 (sqrt), 5 (certified division), 2 (apply)
        cycles = 64 * 166.0 * a.sim_steps
        t_ideal_ms = cycles / (mhz * 1e6) * 1e3
        return {"chain_cycles_per_variant": cycles, "ideal_ms": t_ideal_ms, "frac": t_ideal_ms / kernel_ms,
                "model": "64 serial projections per step x ~166 cycles (binding while <= 1 warp per SMSP, "
                         "n <= 18 944)"}
    if a.model != "box" or ops_exec is None:
        return None
    steps = a.sim_steps
    gnd = max(0.0, (16.0 * n * steps - ops_exec) / (6.0 * n))  # average grounded steps per variant
    cycles = 8.07 * (5.0 * gnd + 6.0 * (steps - gnd))
    t_ideal_ms = cycles / (mhz * 1e6) * 1e3
    return {"chain_cycles_per_variant": cycles, "grounded_steps_per_variant": gnd,
            "ideal_ms": t_ideal_ms, "frac": t_ideal_ms / kernel_ms,
            "model": "5 (grounded) or 6 (otherwise) dependent FP64 ops per step x 8.07 cycles"}


# ---------------------------------------------------------------------- ours
def run_ours(a, ws, rank, local):
    import torch
    import paper_2502_11129_b200 as hb

    dist = None
    local = local % max(1, torch.cuda.device_count())  # >1 rank per GPU only for gloo tests
    torch.cuda.set_device(local)
    backend = os.environ.get("HB_DIST_BACKEND", "nccl")
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    kind = hb.parse_model_kind(a.model)
    if a.workload == "ea":
        return run_ea_bench(a, ws, rank, local, dist, dev, red_dev, kind)

    # Global batch (variants per GPU x N) split by the paper's splitter
    # retargeted to N GPUs: every rank times the same probe on its own GPU
    # (calibrate_ranks), the times are all-gathered, and plan_allocation_n
    # gives each rank a contiguous share in proportion to its throughput.
    n_total = a.variants * ws if a.scaling == "weak" else a.variants
    from paper_2502_11129_b200 import _lib as _hl
    fp32 = a.precision == "fp32"
    ex = hb.GpuExecutor(local, precision=_hl.HB_PRECISION_FP32 if fp32 else _hl.HB_PRECISION_FP64)
    calib = None
    if ws > 1:
        from paper_2502_11129_b200 import distributed as hbd
        calib = hbd.calibrate_ranks(kind, a.sim_steps, max(1, n_total // ws), ex, dist)
        shares = hb.plan_allocation_n(calib, n_total)
    else:
        shares = [n_total]
    begin = sum(shares[:rank])
    seeds = np.arange(begin, begin + shares[rank], dtype=np.uint64)
    n = len(seeds)

    ctx = ex.ctx
    ext = torch.cuda.ExternalStream(ctx.stream, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident kernel timing (value) ----
    ctx.stage(kind, seeds)
    with torch.cuda.stream(ext):
        for _ in range(a.warmup):
            flush.zero_()
            ctx.launch(a.sim_steps)
    ctx.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(a.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(dev)
    ctx.synchronize()
    ops0 = ctx.work_counter() if a.model == "box" else 0
    t0 = time.perf_counter()
    with torch.cuda.stream(ext):
        for e0, e1 in evs:
            flush.zero_()           # L2 flush, outside the event pair
            e0.record(ext)
            ctx.launch(a.sim_steps)
            e1.record(ext)
    ctx.synchronize()
    torch.cuda.synchronize(dev)
    barrier()
    wall_region = time.perf_counter() - t0
    clk = clocks.stop()
    kernel_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    sum_ms = max_over_ranks(sum(kernel_ms))
    ms_per_step = sum_ms / a.steps
    units = n_total * a.sim_steps  # variant-steps per bench step, all ranks
    value = units / (ms_per_step * 1e-3)
    ops_exec = (ctx.work_counter() - ops0) / a.steps if a.model == "box" else None
    out, fail = ctx.fetch()
    assert int(np.sum(fail)) == 0, "blow-up in bench workload"
    _, replays = ctx.last_launch_stats()

    # ---- roofline: FP64 pipe (measured probe on this device) ----
    peak_ops, _ = ctx.fp64_peak()
    if fp32 and a.model != "box":
        # FP32 mode: float-float positions on the FP32 pipe; nominal peak =
        # 148 SMs x 128 FP32 lanes x the SM clock sampled during the run
        peak_ops = 148 * 128 * 1e6 * (clk.get("sm_mhz") or 1965.0)
    per_gpu_rate = n * a.sim_steps / (float(np.mean(kernel_ms)) * 1e-3)
    achieved = W_ALG[a.model] * per_gpu_rate
    traffic = load_traffic(a.model, a.variants, a.sim_steps)
    kmean_s = float(np.mean(kernel_ms)) * 1e-3
    # Box elides the z operations exactly at the grounded fixed point
    # (DESIGN.md §3.1), so SURVEY's W_alg over-counts its work at long
    # horizons (fractions above 1): for Box `achieved` / `frac` are the FP64
    # ops the launch really executed (the kernel's own counter), W_alg beside
    # it.  The multi-body kernels execute every algorithmic op (and more), so
    # W_alg is their (conservative) count.
    exec_rate = None if ops_exec is None else ops_exec / kmean_s
    head = exec_rate if exec_rate is not None else achieved
    roof = {"bound": "fp32" if fp32 and a.model != "box" else "fp64",
            "achieved": head / 1e12, "peak": peak_ops / 1e12,
            "unit": "TFLOP/s", "frac": head / peak_ops, "traffic": traffic,
            "ops_basis": "executed (hb_work_counter)" if exec_rate is not None else "W_alg (SURVEY.md §8d)",
            "achieved_w_alg": achieved / 1e12, "frac_w_alg": achieved / peak_ops,
            "algorithmic_ops_per_variant_step": W_ALG[a.model],
            "peak_source": ("nominal 148 SM x 128 FP32 lanes x sampled SM clock (FP32 mode)"
                            if fp32 and a.model != "box" else
                            "measured on this device by hb_fp64_peak (DMUL+DADD stream, no FMA); "
                            "MEASURED_PEAKS.json has no FP64 figure"),
            "kernel": hb.kernel_name(kind, n),
            "kernel_ms_mean": float(np.mean(kernel_ms)),
            "exact_step_replays": replays,
            # Box elides the z operations exactly at the grounded fixed point
            # (DESIGN.md §3.1): the FP64 work the launch really executed, per
            # the kernel's own counter, and the pipe fraction it implies
            "executed_ops_per_launch": ops_exec,
            "frac_executed": None if exec_rate is None else exec_rate / peak_ops,
            # The bound that actually binds Box at this size: one warp per
            # SMSP, each step a dependent FP64 chain (5 ops grounded, 6 in
            # flight / landing) at the measured 8.07-cycle DADD/DMUL latency
            # (tools/ubench_fp64.cu).  Ideal time = that chain for the average
            # variant's mix of grounded / other steps, at the sampled SM clock.
            "latency_bound": latency_bound(a, n, ops_exec, float(np.mean(kernel_ms)), clk),
            "hbm_bytes_per_launch_algorithmic":
                n * ((0 if a.model == "box" else
                      8 * (6 * BODIES[a.model] + CONS[a.model] + EXTRA_ROWS.get(a.model, 0)))
                     + 8 + 32 + 8)}

    # ---- e2e through the drop-in boundary (host seeds -> host results) ----
    # The reference-facing boundary is the C ABI (include/hbgpu.h) that the
    # C++ adapter hbgpu::gpu_executor wraps: hb_run_batch is timed directly
    # (ctypes, one call per step), with the step's seeds in page-locked host
    # memory and the 32-byte VariantResults landing in a page-locked host
    # buffer; the Python mirror GpuExecutor.run is timed too and reported.
    e2e = None
    if not a.no_e2e:
        import ctypes as C

        from paper_2502_11129_b200 import _lib
        host_seeds = _lib.pinned.empty(n, np.uint64)
        host_seeds[:] = seeds
        host_out = _lib.pinned.empty(n, hb.RESULT_DTYPE)
        wall = C.c_double(0)
        sp, op, h = _lib.ptr(host_seeds), _lib.ptr(host_out), ctx.handle

        def abi_call():
            st = _lib.lib.hb_run_batch(h, int(kind), sp, n, a.sim_steps, op, None, C.byref(wall))
            if st != 0:
                raise RuntimeError(f"hb_run_batch: status {st}")

        def timed(fn):
            for _ in range(a.warmup):
                fn()
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(a.steps):
                fn()
            t = time.perf_counter() - t0
            barrier()
            return max_over_ranks(t)

        t_e2e = timed(abi_call)
        assert np.array_equal(host_out, out)
        req = hb.BatchRequest(kind, host_seeds, a.sim_steps)
        t_py = timed(lambda: ex.run(req))
        assert np.array_equal(ex.run(req).results, out)
        rows = 6 * BODIES[a.model] + CONS[a.model]
        rows += EXTRA_ROWS.get(a.model, 0)
        init_bytes = 0 if a.model == "box" else 8 * rows  # Box initial state is built on the device
        e2e = {"value": units * a.steps / t_e2e, "unit": "variant-steps/s",
               "h2d_bytes_per_step": n_total * (8 + init_bytes),
               "d2h_bytes_per_step": n_total * 32 + 8 * ws,
               "ms_per_step": 1e3 * t_e2e / a.steps,
               "path": "C ABI hb_run_batch (include/hbgpu.h; what hbgpu::gpu_executor::run calls) with "
                       "pinned host seeds and results" + (" (Box: zero-copy: the kernel reads the seeds and "
                                                          "writes the results through the host mapping)"
                                                          if a.model == "box" else
                                                          " (host init + H2D + kernel + D2H)"),
               "python_mirror_ms_per_step": 1e3 * t_py / a.steps}

    # ---- FP32 mode: tolerance and selection agreement vs the FP64 product ----
    fp32_check = None
    if fp32 and rank == 0:
        ex64 = hb.GpuExecutor(local)
        f64 = ex64.run(hb.BatchRequest(kind, seeds, a.sim_steps)).results["fitness"]
        f32 = out["fitness"]
        rel = np.abs(f32 - f64) / np.maximum(np.abs(f64), 1e-3)
        mu = n // 2  # (mu + lambda) parents of this batch as a population (ea.cpp:60-72)
        o32 = np.argsort(-f32, kind="stable")[:mu]
        o64 = np.argsort(-f64, kind="stable")[:mu]
        fp32_check = {"vs": "FP64 product (bit-exact with the reference) on the same seeds",
                      "max_rel_fitness_err": float(rel.max()), "median_rel_fitness_err": float(np.median(rel)),
                      "frac_rel_err_above_1e-4": float(np.mean(rel > 1e-4)),
                      "parent_set_overlap": len(set(o32.tolist()) & set(o64.tolist())) / max(1, mu),
                      "parent_rank_identical_fraction": float(np.mean(o32 == o64)),
                      "stated_tolerance": "tests/test_gpu_fp32.py (DESIGN.md §4.1)"}
        ex64.ctx.close()

    cpu = None
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        try:
            cpu = cpu_reference_rate(int(kind), n, a.sim_steps)
        except Exception as exc:  # noqa: BLE001
            cpu = {"error": str(exc)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "variant-steps/s", "n_gpus": ws,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
                "dtype": "f32 (float-float positions)" if fp32 and a.model != "box" else "f64",
                "data": "synthetic (seeds 0..N-1 through build_model; no datasets)",
                "config": {"workload": workload_name(a), "model": a.model,
                           "variants_per_gpu": n_total // ws if a.scaling == "strong" else a.variants,
                           "global_variants": n_total,
                           "sim_steps": a.sim_steps,
                           "parallelism": f"dp{ws} (independent variants; contiguous slices "
                                          "from plan_allocation_n)",
                           "splitter": ({"calibration_wall_s": calib, "shares": [int(x) for x in shares]}
                                        if calib else None),
                           "l2": "flushed between timed launches (256 MiB write outside the "
                                 "event pair)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "gpu_launches": a.steps, "e2e_gpu_launches": a.steps if e2e else 0,
                "bracket_wall_s": wall_region,
                "parity": ("FP32 mode: within the stated tolerance, see fp32" if fp32 and a.model != "box"
                           else "bit-exact FP64 vs reference")}
        if fp32_check is not None:
            line["fp32"] = fp32_check
        print(json.dumps(line))
    ex.ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def run_ea_bench(a, ws, rank, local, dist, dev, red_dev, kind):
    """configs[4]: the full (mu + lambda) generation loop.  One bench step =
    one run_ea of `--generations` generations over `--population` genomes
    (pop + G * pop/2 variants simulated through `--sim-steps` steps each).
    N = 1: the native device loop (hb_run_ea on one context).
    N > 1: rank 0 drives all N GPUs in process — hb_run_ea over N contexts:
    offspring sharded by the throughput splitter (hb_calibrate: CUDA-event
    probe per GPU, snapped to equal shares for equal GPUs), each GPU fed by
    its persistent worker thread, generations chained by cross-device events
    and the fitness slices gathered into GPU 0 by peer copies over NVLink (no
    host synchronisation per generation for Box); the other ranks only join
    the barrier (their time is 0, so the max over ranks is rank 0's)."""
    import torch
    import paper_2502_11129_b200 as hb
    pop, G = a.population, a.generations
    evaluated = pop + G * (pop // 2)
    if ws > 1:
        # one context per GPU (modulo the visible devices: several ranks per
        # GPU only in the gloo tests)
        ngpu = max(1, torch.cuda.device_count())
        ex = hb.MultiGpuExecutor([d % ngpu for d in range(ws)]) if rank == 0 else None
        calib = ex.calibrate(kind, a.sim_steps, max(1, (pop // 2) // ws)) if rank == 0 else None
    else:
        ex = hb.GpuExecutor(local)
        calib = None

    def one():
        if ex is None:
            return None
        return hb.run_ea(kind, pop, G, a.sim_steps, ex, seed=0)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(a.warmup):
        r = one()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.perf_counter()
    profs = []
    for _ in range(a.steps):
        r = one()
        if r is not None:
            profs.append(r.profile)
    torch.cuda.synchronize(dev)
    t = max_over_ranks(time.perf_counter() - t0 if ex is not None else 0.0)
    clk = clocks.stop()
    value = evaluated * a.sim_steps * a.steps / t
    if rank == 0:
        ev = sum(p.evaluation_s for p in profs)
        tot = sum(p.total_s for p in profs)
        host = sum(p.host_overhead_s for p in profs)
        line = {"metric": METRIC, "value": value, "unit": "variant-steps/s", "n_gpus": ws,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t / a.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (genomes rng::at(seed ^ kInitKey, i), ea.cpp:48-52)",
                "config": {"workload": f"ea: run_ea {a.model} pop {pop} x {G} generations x "
                                       f"{a.sim_steps} steps (BASELINE configs[4])",
                           "model": a.model, "population": pop, "generations": G,
                           "sim_steps": a.sim_steps, "variants_simulated_per_step": evaluated,
                           "parallelism": f"{ws} GPU(s) in one process: offspring shards "
                                          "(plan_allocation_n over hb_calibrate times), per-generation "
                                          "fitness gather by peer copy into GPU 0",
                           "splitter": (None if calib is None else
                                        {"device_times_s": calib[0], "device_ok": calib[1],
                                         "spreads": calib[2]})},
                "e2e": {"value": value, "unit": "variant-steps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 16 * pop,
                        "path": "run_ea -> hb_run_ea (genomes created and selected on GPU 0; "
                                "evaluations sharded over the GPUs; final population D2H)"},
                "evaluation_fraction": ev / tot if tot else None,
                "phases_ms_per_run": {k: 1e3 * sum(getattr(p, k + "_s") for p in profs) / a.steps
                                      for k in ("selection", "evaluation", "bookkeeping", "total",
                                                "host_overhead")},
                "host_overhead_us_per_generation": 1e6 * host / max(1, len(profs)) / (G + 1),
                "best_fitness": r.best_fitness, "clocks": clk,
                # per run: genome init; per evaluation and GPU the simulation
                # (+ the fitness gather, except Box, whose kernel writes
                # fitness; + the state initialiser for multi-body models); per
                # generation the selection (cluster sort, then tie fix +
                # select + offspring in one kernel)
                "gpu_launches": a.steps * (1 + (1 if int(kind) == 0 else 3) * (G + 1) * ws + 2 * G),
                "parity": "genomes + fitness bit-identical to reference run_ea"}
        print(json.dumps(line))
    if ex is not None:
        for c in (ex.ctxs if ws > 1 else [ex.ctx]):
            c.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    a = parse()
    ws, rank, local = dist_env()
    if a.impl == "reference":
        run_reference(a, ws, rank)
        return
    run_ours(a, ws, rank, local)


if __name__ == "__main__":
    main()
