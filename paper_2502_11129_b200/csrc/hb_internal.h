// hb_internal.h — interface between the host runtime (hb_runtime.cpp) and
// the kernels (hb_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/hbgpu.h"
#include "hb_model.h"

namespace hb {

// One batch on one device.
//  init:  SoA rows (state_rows(kind) x ld doubles), read-only; nullptr for
//         Box means "generate the initial state from seeds on the device".
//  seeds: device seeds (n).
//  out:   n x VariantResult (32 B, the reference layout).
//  fail:  n x first failing step (0 = completed).
//  counters: [0] += #failed variants, [1] += #exact step replays.
//  final_state (nullable): SoA rows, ld.
// Loop-invariant step coefficients (hoisting them is value-preserving;
// SURVEY.md §8 a3): computed on the host per launch and passed in the kernel
// parameters, so the stepping kernels read them as constant-bank operands
// instead of holding six doubles in registers for the whole horizon.
struct StepCoefs {
    double dt, gdt, damp, inv_dt, half_k_stiff, half_k_soft;
};

HB_HD StepCoefs step_coefs(double dt) {
    StepCoefs c{};
    c.dt = dt;
    c.gdt = kGravity * dt;          // v.z -= kGravity * dt        (simkernel.cpp:130)
    c.damp = 1.0 - kDamping * dt;   // damp = 1 - damping * dt     (:126)
    c.inv_dt = 1.0 / dt;            // (:156)
    const double ks = (kStiffLink * dt) * dt;  // c.stiffness * dt * dt (:145)
    const double kf = (kSoftLink * dt) * dt;
    c.half_k_stiff = 0.5 * (ks < 1.0 ? ks : 1.0);  // std::min(1.0, x), then 0.5 * k (:146)
    c.half_k_soft = 0.5 * (kf < 1.0 ? kf : 1.0);
    return c;
}

struct SimArgs {
    const double* init;
    const uint64_t* seeds;
    size_t n;
    size_t ld;
    uint64_t steps;
    double dt;
    hb_variant_result* out;
    uint64_t* fail;
    unsigned* counters;
    double* final_state;
    // nullable: host-mapped flag a failing variant sets to 1 (plain store;
    // lets a zero-copy launch report "something blew up" without a D2H)
    volatile unsigned* fail_flag;
    // nullable (Box): running total of the algorithmic FP64 ops the launch
    // executed — 16 per variant-step, 10 for steps run at the grounded fixed
    // point (z elided exactly); hb_work_counter reads it
    unsigned long long* ops;
    // nullable (Box): write each variant's fitness (0 for a failed one) here
    // instead of the VariantResult records — the generation loop's
    // evaluation, which needs nothing else
    double* fitness = nullptr;
    // step_coefs(dt), filled by launch_sim for the multi-body kernels
    StepCoefs k{};
};

cudaError_t launch_sim(int kind, const SimArgs& a, cudaStream_t st, int sms, int variant);
// Initial SoA state rows (state_rows(kind) x n, row stride n) of a
// multi-body kind from the seeds and the host's cos / sin rows
// (2 init_angles(kind) x n): hb_init.cu.
cudaError_t launch_init(int kind, const uint64_t* seeds, const double* trig, size_t n, double* soa,
                        cudaStream_t st);
// The Box stepping launch through a per-context one-node CUDA graph whose
// kernel parameters are updated in place when they change: cheaper on the
// host and on the device than a plain launch (the drop-in call's fixed cost).
struct BoxGraph {
    cudaGraph_t graph[2] = {nullptr, nullptr};  // [from seeds, from states]
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    cudaGraphNode_t node[2] = {nullptr, nullptr};
    SimArgs last[2];              // the parameters the instantiated node holds
    unsigned last_block[2] = {0, 0};
};
cudaError_t launch_box_graph(BoxGraph& g, const SimArgs& a, cudaStream_t st, int sms);
void destroy_box_graph(BoxGraph& g);
const char* kernel_name(int kind, size_t n, int variant);
// FP32 throughput mode (hb_fp32.cu; HB_PRECISION_FP32): host-built states only
cudaError_t launch_sim_fp32(int kind, const SimArgs& a, cudaStream_t st);
const char* kernel_name_fp32(int kind);
cudaError_t launch_fp64_probe(double* scratch, int sms, int iters, cudaStream_t st, double* ops);
cudaError_t launch_fastpath_check(const double* x, const double* y, size_t n, double* o0, double* o1,
                                  double* o2, double* o3, unsigned char* flags, cudaStream_t st);

// Generation loop helpers (hb_ea.cu).
// g_dev (optional): the graph-replayed loop's generation counter, reset to 0
// (each selection graph's first kernel advances it)
cudaError_t ea_init_genomes(uint64_t seed, size_t pop, uint64_t* d_genomes, cudaStream_t st,
                            uint64_t* g_dev = nullptr);
cudaError_t ea_fitness_from_results(const hb_variant_result* out, size_t n, double* fitness,
                                    cudaStream_t st);
size_t ea_select_scratch_bytes(size_t pop);
cudaError_t ea_select_vary(const uint64_t* d_genomes, const double* d_fitness, size_t pop, uint64_t g,
                           uint64_t* d_next, double* d_next_fit, void* scratch, size_t scratch_bytes,
                           cudaStream_t st);
cudaError_t ea_select_vary_graph(const uint64_t* d_genomes, const double* d_fitness, size_t pop,
                                 uint64_t* g_dev, uint64_t* d_next, double* d_next_fit, void* scratch,
                                 size_t scratch_bytes, cudaStream_t st, cudaGraphExec_t* exec);

}  // namespace hb
