/*
 * hbgpu.h — C ABI of the B200-native batched variant-simulation backend.
 *
 * This is the drop-in boundary for the reference's accelerator slot
 * (/root/reference/proj):
 *
 *   hetbench::batch_executor::run(const BatchRequest&) -> BatchResult
 *       include/hetbench/executor.hpp:68-73
 *   currently filled by synthetic_executor::run     src/executor.cpp:137-170
 *   per variant: simulate(kind, seed, steps)         src/simkernel.cpp:187-203
 *
 * A reference-side adapter (include/hbgpu/hetbench_gpu_executor.hpp, shown in
 * INTEGRATION.md) derives from hetbench::batch_executor and forwards run()
 * to hb_run_batch(); nothing else in the reference changes.
 *
 * Rules: plain C types only; no exception crosses this boundary; every call
 * returns an hb_status and the context keeps the last error message.  One
 * context per device; a context is single-threaded (callers serialise per
 * context), distinct contexts may be driven from distinct host threads
 * concurrently (run_hybrid runs the accelerator share on a helper
 * std::thread, src/scheduler.cpp:148-153).  There is no CPU fallback: on a
 * host without a usable sm_100 device hb_ctx_create fails with
 * HB_NO_DEVICE.
 */
#ifndef HBGPU_H
#define HBGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HBGPU_ABI_VERSION 2

/* hetbench::ModelKind (include/hetbench/simkernel.hpp:14) — same ordinals.
 * HB_CPG_HINGE (4) is NOT a reference model: the "Revolve2-style modular
 * robot with hinge joints + CPG controller" of BASELINE configs[2] (SPEC.md:101
 * leaves it undefined); its definition and only oracle is oracle/hb_oracle.c
 * (hbo_cpg_*).  Every entry point taking a `kind` accepts 0..4. */
typedef enum {
    HB_BOX = 0,
    HB_BOX_AND_BALL = 1,
    HB_ARM_WITH_ROPE = 2,
    HB_HUMANOID = 3,
    HB_CPG_HINGE = 4
} hb_model_kind;

typedef enum {
    HB_OK = 0,
    HB_INVALID_ARG = 1,    /* std::invalid_argument in the reference (executor.cpp:60-65) */
    HB_CUDA_ERROR = 2,     /* device/runtime failure: the back-end is dead to calibrate() */
    HB_BLOWUP_PARTIAL = 3, /* some variants blew up; the rest completed (batch_failure) */
    HB_NO_DEVICE = 4       /* no usable sm_100 device */
} hb_status;

/* Byte-for-byte hetbench::VariantResult (simkernel.hpp:51-58): 32 B POD. */
typedef struct {
    uint64_t seed;
    double fitness;
    uint64_t checksum;
    uint64_t steps_executed;
} hb_variant_result;

/* hetbench::AllocationPlan (scheduler.hpp:24-30). */
typedef struct {
    uint64_t n_total;
    uint64_t n_cpu;
    uint64_t n_accel;
    double accel_fraction;
    double requested_accel_fraction;
} hb_allocation_plan;

typedef struct hb_ctx hb_ctx;

/* ---- library / model introspection ------------------------------------- */
int hb_abi_version(void);
/* Number of CUDA devices visible (0 when none / driver missing). */
int hb_device_count(void);
/* body_count (simkernel.hpp:23-31) and the constraint count of build_model
 * (simkernel.cpp:95-118); -1 for an unknown kind. */
int hb_body_count(int kind);
int hb_constraint_count(int kind);
/* Rows of the structure-of-arrays state for `kind`: 3n positions (body-major,
 * x,y,z), 3n velocities, m rest lengths.  Row r of variant i lives at
 * soa[r * ld + i]. */
int hb_state_rows(int kind);
/* Last error of calls that have no context (thread-local). */
const char* hb_global_error(void);

/* ---- context -------------------------------------------------------------- */
hb_status hb_ctx_create(int device, hb_ctx** out);
void hb_ctx_destroy(hb_ctx* ctx);
const char* hb_last_error(const hb_ctx* ctx);
int hb_ctx_device(const hb_ctx* ctx);
/* The cudaStream_t every launch of this context is issued on. */
void* hb_ctx_stream(hb_ctx* ctx);
/* Host threads used for the host side of initialisation — the libm
 * cos / sin of build_model's body angles (the rest of the multi-body state
 * is built on the device; the generic kernel variant builds all of it on
 * the host) — and for staging copies (default: all hardware threads,
 * capped at 64). 0 = default. */
hb_status hb_ctx_set_host_threads(hb_ctx* ctx, int threads);

/* Kernel family used by this context.  HB_KERNEL_AUTO (default) = the
 * optimised kernels (branch-free projection with exact replay, two-lane
 * humanoid, device-side Box init); HB_KERNEL_GENERIC = the plain
 * reference-order kernel (library sqrt / '/', every branch), kept as an
 * in-tree cross-check.  Both are bit-exact with simulate(). */
#define HB_KERNEL_AUTO 0
#define HB_KERNEL_GENERIC 1
hb_status hb_ctx_set_kernel(hb_ctx* ctx, int variant);

/* Arithmetic of this context's stepping kernels.  HB_PRECISION_FP64
 * (default) = the product path, bit-exact with simulate() (FP64 in the
 * reference's operation order).  HB_PRECISION_FP32 = the FP32 throughput
 * mode of SURVEY.md §8 row f3 for the multi-body models: float-float
 * positions, FP32 increments, FMA-compensated constants, MUFU rsqrt; NOT
 * bit-exact — fitness within the tolerance stated in tests/test_gpu_fp32.py,
 * checksums of this mode's own state; the same initial states.  Box keeps
 * the (faster) bit-exact FP64 kernel in either mode. */
#define HB_PRECISION_FP64 0
#define HB_PRECISION_FP32 1
hb_status hb_ctx_set_precision(hb_ctx* ctx, int precision);

/* Zero-copy Box path (default on): when a Box batch's seeds and `out` are both
 * mapped page-locked memory (e.g. hb_host_alloc), the kernel reads the seeds
 * and writes the results through the host mapping — no H2D / D2H operation
 * on the call's critical path.  0 disables it (always stage + DMA). */
hb_status hb_ctx_set_zero_copy(hb_ctx* ctx, int enable);

/* ---- utilisation trace (BatchResult::utilization_trace, executor.hpp:26-35)
 * With the monitor on, every hb_run_batch on this context records a trace:
 * NVML GPU utilisation (nvmlDeviceGetUtilizationRates, the driver's
 * libnvidia-ml.so.1 loaded at run time; absent NVML = no such samples) at
 * 20 Hz while the call runs, t in seconds since the call started, then one
 * final synchronised sample at t = the call's wall time: the share of the
 * wall time during which the stepping kernel ran (CUDA events around the
 * launch) — the quantity NVML reports, exact for this call however short.
 * Off by default (it adds two event records and a sampler hand-off). */
typedef struct {
    double t;             /* seconds since the call started */
    double accel_percent; /* [0, 100] */
} hb_util_sample;
hb_status hb_ctx_set_monitor(hb_ctx* ctx, int enable);
/* Samples of the last monitored hb_run_batch: *count = their number; the
 * first min(cap, *count) are copied to out (nullable). */
hb_status hb_last_utilization(const hb_ctx* ctx, hb_util_sample* out, size_t cap, size_t* count);

/* Fault injection (test seam; the counterpart of the reference's
 * simulate_fn seam, executor.hpp:89-90, that its tests use to make a back-end
 * throw).  Applies to hb_run_batch calls on this context until reset:
 *   HB_FAULT_NONE    no injection (default);
 *   HB_FAULT_BLOWUP  every variant whose seed == `seed` is reported as blown
 *                    up at step 1 (fail_step 1, record {seed, 0, 0, 1},
 *                    HB_BLOWUP_PARTIAL) — the batch_failure path;
 *   HB_FAULT_DEVICE  every call fails with HB_CUDA_ERROR, as a dead device —
 *                    the path on which calibrate / run_hybrid treat a
 *                    back-end as failed (scheduler.cpp:40-49,162-183). */
#define HB_FAULT_NONE 0
#define HB_FAULT_BLOWUP 1
#define HB_FAULT_DEVICE 2
hb_status hb_ctx_inject_fault(hb_ctx* ctx, int mode, uint64_t seed);

/* Start-up reservation: size every device and pinned staging buffer for
 * batches of up to `n` variants of `kind` and load the kernel such a batch
 * runs (one discarded 1-step batch of seeds 0..n-1).  A context's first call
 * at a new size otherwise pays its allocations and the lazy kernel load in
 * its wall_time_s (tools/cold_probe.py: 17-85 ms against 0.5-12 ms warm at
 * the sweep sizes), which a single-probe calibrate (scheduler.cpp:30-56)
 * reads as accelerator speed.  Optional; hb_run_batch grows on demand. */
hb_status hb_ctx_reserve(hb_ctx* ctx, int kind, size_t n);

/* Page-locked host memory (cudaHostAlloc, portable + mapped).  hb_run_batch / hb_fetch
 * DMA the results straight into an `out` buffer allocated here (no staging
 * copy); any other buffer goes through the context's staging buffer. */
void* hb_host_alloc(size_t bytes);
void hb_host_free(void* ptr);

/* Failure steps of the last fetched batch (n entries; 0 = completed), for
 * callers that passed fail_step = NULL and got HB_BLOWUP_PARTIAL. */
hb_status hb_last_fail_steps(hb_ctx* ctx, uint64_t* fail_step, size_t n);

/* Counters of the last fetched batch: variants that blew up, and steps the
 * optimised kernels recomputed on the exact (library sqrt / div) path
 * because a fast-path guard fired (0 in normal operation).  After several
 * hb_launch calls without an intervening fetch they are sums over those
 * launches (the per-variant results are always the last launch's). */
hb_status hb_last_launch_stats(hb_ctx* ctx, uint64_t* failed, uint64_t* exact_replays);

/* Running total of the algorithmic FP64 operations this context's Box
 * launches executed (16 per variant-step; 10 for the steps a
 * warp ran at the exact grounded fixed point (p.z, v.z) = (+0, +0), whose z
 * operations are elided; steps up to the failing one for a blown-up
 * variant).  Read the difference around the launches of interest; it
 * synchronises the context's stream.  Other models: W_alg x variant-steps. */
hb_status hb_work_counter(hb_ctx* ctx, uint64_t* ops);

/* ---- the drop-in call ------------------------------------------------------
 * batch_executor::run (executor.hpp:70) for `n` seeds through `steps` fixed
 * dt = kSimDt steps.  out[i] is the VariantResult of seeds[i] (seed order);
 * fail_step[i] = 0 when variant i completed, otherwise the 1-based step whose
 * end-of-step check raised numerical_blowup (simkernel.cpp:165-169), and
 * out[i] is then unspecified.  Returns HB_BLOWUP_PARTIAL when any variant
 * failed.  *wall_time_s (nullable) = steady-clock seconds around the whole
 * call including host init, H2D and D2H (executor.cpp:91-115 semantics).
 * fail_step may be NULL only if the caller does not need failure detail. */
hb_status hb_run_batch(hb_ctx* ctx, int kind, const uint64_t* seeds, size_t n, uint64_t steps,
                       hb_variant_result* out, uint64_t* fail_step, double* wall_time_s);

/* Host-side initialiser: build_model (simkernel.cpp:59-120) for each seed,
 * written as SoA rows (hb_state_rows(kind) rows, leading dimension ld >= n). */
hb_status hb_build_states(int kind, const uint64_t* seeds, size_t n, double* soa, size_t ld);

/* Run from caller-supplied initial states (host SoA, ld = n) with step size
 * dt (> 0, else HB_INVALID_ARG as step() throws at simkernel.cpp:123).
 * seeds (nullable) only fill out[i].seed.  final_soa (nullable, ld = n)
 * receives the final positions/velocities rows (rest rows copied through). */
hb_status hb_run_states(hb_ctx* ctx, int kind, const double* init_soa, size_t n, uint64_t steps,
                        double dt, const uint64_t* seeds, hb_variant_result* out,
                        uint64_t* fail_step, double* final_soa);

/* ---- device-resident (staged) path used for kernel-only timing ------------
 * hb_stage: host init + H2D into the context's device buffers (synchronous).
 * hb_launch: enqueue one stepping kernel over the staged batch on the
 *   context stream (asynchronous; the staged inputs are not modified, so it
 *   can be re-launched).
 * hb_fetch: D2H of the last launch's results (synchronous). */
hb_status hb_stage(hb_ctx* ctx, int kind, const uint64_t* seeds, size_t n);
hb_status hb_launch(hb_ctx* ctx, uint64_t steps);
hb_status hb_synchronize(hb_ctx* ctx);
hb_status hb_fetch(hb_ctx* ctx, hb_variant_result* out, uint64_t* fail_step);
/* Kernel variant the dispatcher picks for (kind, n): written to buf. */
hb_status hb_kernel_name(int kind, size_t n, char* buf, size_t cap);

/* ---- failure messages ------------------------------------------------------
 * The what() of the numerical_blowup simulate() re-throws
 * (simkernel.cpp:167-168,194):
 *   "coordinate left the stable regime at t=<std::to_string(time)> (seed S)"
 * where time is the FP64 running sum of dt after fail_step steps. */
int hb_format_blowup(uint64_t seed, uint64_t fail_step, double dt, char* buf, size_t cap);

/* ---- splitter (paper §6, scheduler.cpp:58-87) ----------------------------
 * plan_allocation bit-for-bit (n_total >= 1). */
hb_status hb_plan_allocation(double t_cpu_s, double t_accel_s, int cpu_ok, int accel_ok,
                             uint64_t n_total, hb_allocation_plan* out);
/* N-way "peeling" generalisation across `count` back-ends with calibrated
 * probe times t_s[d] (ok[d] = 0 marks a dead back-end): for d = count-1..1,
 * share[d] = plan_allocation({t_cpu = T_rest, t_accel = t_s[d]}, remaining)
 * .n_accel, T_rest = t_s[0] when only back-end 0 remains, else
 * 1 / sum_{j<d} 1/t_s[j]; back-end 0 takes the remainder.  For count == 2
 * this is plan_allocation exactly (shares[0] = n_cpu, shares[1] = n_accel). */
hb_status hb_plan_allocation_n(const double* t_s, const int* ok, int count, uint64_t n_total,
                               uint64_t* shares);

/* ---- multi-device executor -------------------------------------------------
 * One context and one persistent host thread per device; the batch is cut
 * into contiguous slices (shares[d] variants to device d, in device order, as
 * run_hybrid slices seeds at scheduler.cpp:122-127) and merged in seed order.
 * shares == NULL splits evenly.  per_device_wall_s (nullable, `count`
 * entries) receives each device's run wall time.
 * Degraded mode (the N-way form of run_hybrid's re-dispatch,
 * scheduler.cpp:162-183): a device whose slice fails with anything but
 * HB_BLOWUP_PARTIAL is dead for the rest of the call and its slice is
 * re-planned over the surviving devices with hb_plan_allocation_n (ok = 0 for
 * the dead ones, the survivors weighted by their original shares); the
 * results are complete and identical to a healthy run.  device_ok (nullable,
 * `count` entries) = 1 for devices that finished their work, *degraded
 * (nullable) = 1 if any device died.  Only when every device fails does the
 * call fail (with the first device's status). */
hb_status hb_run_batch_multi(hb_ctx* const* ctxs, int count, const uint64_t* shares, int kind,
                             const uint64_t* seeds, size_t n, uint64_t steps,
                             hb_variant_result* out, uint64_t* fail_step,
                             double* per_device_wall_s, double* wall_time_s,
                             int* device_ok, int* degraded);

/* ---- calibration (the paper's calibrate step, scheduler.cpp:30-56, on
 * devices) ------------------------------------------------------------------
 * Times the probe batch (seeds 0..probe_n-1 of `kind` through `steps` steps)
 * on every context concurrently with CUDA events on the context's stream:
 * the probe is relaunched back to back until one sample spans >= 5 ms, and
 * t_s[d] is the median per-launch time of `repeats` (>= 1; 5 recommended)
 * such samples, spread[d] (nullable) their relative range (max - min) /
 * median.  A device whose probe fails gets ok[d] = 0 and t_s[d] = 0 (dead to
 * the splitter, like a throwing back-end in calibrate); HB_INVALID_ARG only
 * for bad arguments, otherwise HB_OK if at least one device survived. */
hb_status hb_calibrate(hb_ctx* const* ctxs, int count, int kind, uint64_t probe_n, uint64_t steps,
                       int repeats, double* t_s, double* spread, int* ok);
/* Equal devices get equal shares: if the alive devices' times agree within
 * max(their largest measured spread, min_rel_tol) (relative to the fastest),
 * every alive device's time becomes their mean, so plan_allocation_n splits
 * evenly instead of amplifying measurement noise; otherwise the times are
 * returned unchanged.  Returns 1 if it snapped.  ok / spread nullable. */
int hb_snap_equal_times(const double* t_s, const double* spread, const int* ok, int count,
                        double min_rel_tol, double* out_t_s);

/* ---- FP64 pipe peak probe (roofline denominator) ---------------------------
 * Times a dependent-chain-free DADD/DMUL stream on the context's device and
 * returns the sustained non-FMA FP64 op rate (ops/s) and the kernel time. */
hb_status hb_fp64_peak(hb_ctx* ctx, double* ops_per_s, double* ms);

/* ---- (mu + lambda) generation loop (ea.cpp:33-105) ------------------------
 * run_ea with every generation's evaluation, selection (stable descending
 * sort of fitness) and variation on the devices; only the per-generation
 * fitness of each device's offspring slice crosses to device 0 (peer copy
 * over NVLink) and, for the multi-body models, the offspring seeds go to the
 * host for the libm cos / sin rows of their initial states.  With one
 * context and Box the whole loop is queued without a host round trip per
 * generation (one failure check at the end; a blow-up re-runs the loop with
 * a check per generation to report it).  Offspring are sharded over the
 * `count` contexts by hb_plan_allocation_n(device_times) (NULL = equal).
 * Outputs (host): final population genomes / fitness (pop each, parents ++
 * offspring), best fitness, phase profile; history_* (nullable) receive the
 * population after every generation ((generations + 1) x pop).  Genomes and
 * fitness are bit-identical to the reference run_ea over cpu_executor.
 * A blow-up aborts with HB_BLOWUP_PARTIAL and a batch_failure-style message,
 * as evaluate() throwing aborts run_ea. */
typedef struct {
    double selection_s;
    double variation_s;
    double evaluation_s;
    double bookkeeping_s;
    double total_s;
    /* wall time of the call not covered by device work (first launch
     * latency, enqueue stalls, host round trips, final sync and copies):
     * total_s minus the device span of the loop, where a device span was
     * measured (the queued loops), else 0 */
    double host_overhead_s;
} hb_phase_profile;

hb_status hb_run_ea(hb_ctx* const* ctxs, int count, const double* device_times, int kind, size_t pop,
                    uint64_t generations, uint64_t steps, uint64_t seed, uint64_t* genomes_out,
                    double* fitness_out, double* best_out, hb_phase_profile* profile,
                    uint64_t* history_genomes, double* history_fitness);

/* Device-pointer building blocks of the loop, for callers that keep the
 * population in their own device memory (e.g. torch tensors; one rank per
 * GPU with an NCCL fitness all-gather between them).  All run on the
 * context's stream.
 *   hb_eval_device: simulate d_seeds[0, n) (device) -> d_fitness (device);
 *     synchronises; *n_failed = blown-up variants (HB_BLOWUP_PARTIAL if > 0).
 *   hb_ea_init_genomes: d_genomes[i] = rng::at(seed ^ kInitKey, i).
 *   hb_ea_select_vary: stable descending selection of the top pop/2 and
 *     their offspring for generation g: d_next = parents ++ offspring,
 *     d_next_fitness[0, pop/2) = parent fitness. */
hb_status hb_eval_device(hb_ctx* ctx, int kind, const uint64_t* d_seeds, size_t n, uint64_t steps,
                         double* d_fitness, uint64_t* n_failed);
hb_status hb_ea_init_genomes(hb_ctx* ctx, uint64_t seed, size_t pop, uint64_t* d_genomes);
hb_status hb_ea_select_vary(hb_ctx* ctx, const uint64_t* d_genomes, const double* d_fitness,
                            size_t pop, uint64_t g, uint64_t* d_next, double* d_next_fitness);

/* ---- fast-path self test ----------------------------------------------------
 * Evaluates the kernels' branch-free sqrt(x[i]) replica and their certified
 * division x[i] / RN(sqrt(y[i]^2)) (the reciprocal taken from the sqrt's
 * refined rsqrt, as in the projection) against the library IEEE versions on
 * the device.  Counts operands where the fast path claims validity but
 * differs in any bit (must be 0), and operands it flags for exact replay. */
hb_status hb_check_fast_math(hb_ctx* ctx, const double* x, const double* y, size_t n,
                             uint64_t* sqrt_mismatch, uint64_t* div_mismatch,
                             uint64_t* sqrt_flagged, uint64_t* div_flagged);

#ifdef __cplusplus
}
#endif
#endif /* HBGPU_H */
