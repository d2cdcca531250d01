// hb_fp32.cu — FP32 throughput mode for the
// multi-body models (Box keeps the FP64 kernel in every mode).  NOT bit-exact:
// the product path is the FP64 kernel family in hb_kernels.cu; this mode is
// opt-in per context (hb_ctx_set_precision(ctx, HB_PRECISION_FP32)) and is
// checked against the FP64 oracle within a stated relative tolerance
// (tests/test_gpu_fp32.py), with its EA selection agreement reported.
//
// Why plain FP32 fails and what this does instead.  SURVEY.md §0-2 measured a
// naive FP32 step() at 7.5 % (box, 5 000 steps) to 19 % (arm, 1 000 steps)
// fitness error: positions ~1 m absorb per-step increments ~1e-3 m, so every
// p + v*dt drops ~2^-24 / 2e-3 of the increment, systematically.  Here
//   * positions and predictions are float-float pairs (hi + lo, ~2^-48),
//     so increments are never quantised against the position;
//   * velocities, distances, corrections are FP32 (relative 2^-24, unbiased
//     round-to-nearest: a random walk, not a drift);
//   * the constants whose float rounding would bias every step (damp, dt,
//     g*dt, rest lengths) enter as float-float through FMA-compensated
//     products: v*damp and w*dt carry the FP64 constants' value, so neither
//     (1 - 0.8 dt) nor dt * (1/dt) drifts (RN32(0.002) * 500 = 1 + 4.7e-8
//     would otherwise compound to 1e-3 over 20 000 steps);
//   * correction increments accumulate into the lo word within a step and
//     the pair is renormalised once per step (two_sum).
// Operation order follows step() (simkernel.cpp:122-170): gravity, damping,
// prediction, 8 Gauss-Seidel sweeps in list order with the ground clamp,
// velocity from displacement, contact, blow-up check at |x| <= 1e6.  Fitness
// and the FNV-1a checksum are computed from the FP64 value of the final
// state (hi + lo is exact in double), so results keep the VariantResult
// layout; the checksum is of this mode's state, not the reference's.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hb_device.cuh"
#include "hb_internal.h"
#include "hb_model.h"

namespace hb {

namespace {

struct FF {
    float hi, lo;
};

__device__ __forceinline__ FF ff_of(double x) {
    FF r;
    r.hi = __double2float_rn(x);
    r.lo = __double2float_rn(x - static_cast<double>(r.hi));
    return r;
}

__device__ __forceinline__ double ff_value(const FF& a) {
    return static_cast<double>(a.hi) + static_cast<double>(a.lo);
}

// Knuth two_sum: s + e == a + b exactly.
__device__ __forceinline__ FF two_sum(float a, float b) {
    const float s = __fadd_rn(a, b);
    const float bb = __fsub_rn(s, a);
    const float e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
    return FF{s, e};
}

// a * (C.hi + C.lo) as a pair: exact product of a and C.hi plus a * C.lo.
__device__ __forceinline__ FF mul_ff(float a, const FF& c) {
    const float p = __fmul_rn(a, c.hi);
    const float e = __fmaf_rn(a, c.hi, -p);
    return FF{p, __fmaf_rn(a, c.lo, e)};
}

// RN32(a * (C.hi + C.lo)): one rounding of the compensated product.
__device__ __forceinline__ float mul_c(float a, const FF& c) {
    return __fmaf_rn(a, c.hi, __fmul_rn(a, c.lo));
}

// (a - b) of two pairs, rounded to float (the hi words are close, so their
// difference is exact).
__device__ __forceinline__ float diff_f(const FF& a, const FF& b) {
    return __fadd_rn(__fsub_rn(a.hi, b.hi), __fsub_rn(a.lo, b.lo));
}

// sign of hi + lo (RN keeps the sign of a nonzero sum; 0 only when exact)
__device__ __forceinline__ float ff_sum_f(const FF& a) { return __fadd_rn(a.hi, a.lo); }

struct CoefsF {
    FF damp, dt, gdt;
    float inv_dt, half_k_stiff, half_k_soft;
};

template <int K>
__global__ void __launch_bounds__(64) ff_kernel(SimArgs a) {
    constexpr int n = bodies(K);
    constexpr int m = constraints(K);
    constexpr int R = 3 * n;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= a.n) return;
    const size_t ld = a.ld;
    const double* __restrict__ src = a.init + i;
    FF p[R], q[R];
    float v[R];
    FF rest[m > 0 ? m : 1];
    double rest_d[m > 0 ? m : 1], rcur[m > 0 ? m : 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        p[r] = ff_of(__ldg(src + r * ld));
        v[r] = __double2float_rn(__ldg(src + (R + r) * ld));
    }
#pragma unroll
    for (int c = 0; c < m; ++c) {
        rest_d[c] = __ldg(src + (2 * R + c) * ld);
        rcur[c] = rest_d[c];
        rest[c] = ff_of(rest_d[c]);
    }
    Cpg cpg;
    if constexpr (K == CpgHinge) cpg_load(cpg, src + (2 * R + m) * ld, ld);
    const Coefs k = make_coefs(a.dt);
    CoefsF f;
    f.damp = ff_of(k.damp);
    f.dt = ff_of(k.dt);
    f.gdt = ff_of(k.gdt);
    f.inv_dt = __double2float_rn(k.inv_dt);
    f.half_k_stiff = __double2float_rn(k.half_k_stiff);
    f.half_k_soft = __double2float_rn(k.half_k_soft);
    const double sx = ff_value(p[0]), sy = ff_value(p[1]);
    uint64_t fail = 0;

    for (uint64_t s = 0; s < a.steps; ++s) {
        if constexpr (K == CpgHinge) {
            cpg_update(cpg, k.dt, rest_d + 8, rcur + 8);
#pragma unroll
            for (int l = 0; l < 4; ++l) rest[8 + l] = ff_of(rcur[8 + l]);
        }
        // gravity, damping, prediction (:127-136)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float vv = v[r];
            if (r % 3 == 2) vv = __fsub_rn(__fsub_rn(vv, f.gdt.hi), f.gdt.lo);
            const float w = mul_c(vv, f.damp);
            const FF d = mul_ff(w, f.dt);
            const FF t = two_sum(p[r].hi, d.hi);
            q[r] = FF{t.hi, __fadd_rn(t.lo, __fadd_rn(p[r].lo, d.lo))};
        }
        // 8 Gauss-Seidel sweeps in list order, ground clamp after each
        // (:140-152).  Branch-free and fully unrolled (humanoid: one sweep per
        // trip, registers), so ptxas sees the whole dependency DAG and
        // overlaps independent links across sweeps (the wavefront) itself.
        // dist and 1/dist come from one MUFU rsqrt (~2 ulp: inside this
        // mode's tolerance); the degenerate link (dist < 1e-12, :144) is
        // masked to a zero correction instead of skipped.
#pragma unroll (K == Humanoid ? 1 : kIters)
        for (int it = 0; it < kIters; ++it) {
#pragma unroll
            for (int c = 0; c < m; ++c) {
                const int A = con_a(K, c), B = con_b(K, c);
                const float dx = diff_f(q[3 * B], q[3 * A]);
                const float dy = diff_f(q[3 * B + 1], q[3 * A + 1]);
                const float dz = diff_f(q[3 * B + 2], q[3 * A + 2]);
                const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
                const float inv = rsqrtf(d2);
                const float dist = __fmul_rn(d2, inv);
                const float hk = con_soft(K, c) ? f.half_k_soft : f.half_k_stiff;
                const float stretch = __fsub_rn(__fsub_rn(dist, rest[c].hi), rest[c].lo);
                const float corr = d2 > 1e-24f ? __fmul_rn(__fmul_rn(hk, stretch), inv) : 0.0f;
                const float ex = __fmul_rn(dx, corr), ey = __fmul_rn(dy, corr), ez = __fmul_rn(dz, corr);
                q[3 * A].lo = __fadd_rn(q[3 * A].lo, ex);
                q[3 * A + 1].lo = __fadd_rn(q[3 * A + 1].lo, ey);
                q[3 * A + 2].lo = __fadd_rn(q[3 * A + 2].lo, ez);
                q[3 * B].lo = __fsub_rn(q[3 * B].lo, ex);
                q[3 * B + 1].lo = __fsub_rn(q[3 * B + 1].lo, ey);
                q[3 * B + 2].lo = __fsub_rn(q[3 * B + 2].lo, ez);
            }
#pragma unroll
            for (int b = 0; b < n; ++b)
                if (ff_sum_f(q[3 * b + 2]) < 0.0f) q[3 * b + 2] = FF{0.0f, 0.0f};
        }
        // velocity from displacement, contact, blow-up (:156-169)
        bool ok = true;
#pragma unroll
        for (int b = 0; b < n; ++b) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int r = 3 * b + c;
                v[r] = __fmul_rn(diff_f(q[r], p[r]), f.inv_dt);
                p[r] = two_sum(q[r].hi, q[r].lo);
            }
            if (ff_sum_f(p[3 * b + 2]) <= 0.0f && v[3 * b + 2] < 0.0f) v[3 * b + 2] = 0.0f;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                ok = ok && fabsf(p[3 * b + c].hi) <= 1e6f && fabsf(v[3 * b + c]) <= 1e6f;
        }
        if (!ok) {
            fail = s + 1;
            break;
        }
    }
    uint64_t h = kFnvOffset;
    double fit = 0.0;
    if (fail == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) h = absorb(h, ff_value(p[r]));
#pragma unroll
        for (int r = 0; r < R; ++r) h = absorb(h, static_cast<double>(v[r]));
        if constexpr (K == CpgHinge) {
#pragma unroll
            for (int l = 0; l < 4; ++l) h = absorb(h, cpg.x[l]);
#pragma unroll
            for (int l = 0; l < 4; ++l) h = absorb(h, cpg.y[l]);
        }
        const double dx = ff_value(p[0]) - sx, dy = ff_value(p[1]) - sy;
        fit = sqrt(dx * dx + dy * dy);
    }
    emit(a, i, fit, h, fail);
    if (a.final_state) {
        double* dst = a.final_state + i;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            dst[r * ld] = ff_value(p[r]);
            dst[(R + r) * ld] = static_cast<double>(v[r]);
        }
#pragma unroll
        for (int c = 0; c < m; ++c) dst[(2 * R + c) * ld] = rest_d[c];
        if constexpr (K == CpgHinge) {
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                dst[(2 * R + m + l) * ld] = cpg.x[l];
                dst[(2 * R + m + 4 + l) * ld] = cpg.y[l];
                dst[(2 * R + m + 8 + l) * ld] = cpg.w[l];
                dst[(2 * R + m + 12 + l) * ld] = cpg.c[l];
            }
        }
    }
}

template <int K>
cudaError_t launch_ff(const SimArgs& a, cudaStream_t st) {
    constexpr int kBlock = 64;
    const unsigned grid = static_cast<unsigned>((a.n + kBlock - 1) / kBlock);
    ff_kernel<K><<<grid, kBlock, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_sim_fp32(int kind, const SimArgs& a, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    if (a.init == nullptr) return cudaErrorInvalidValue;  // this mode always takes host-built states
    switch (kind) {
        case Box: return launch_ff<Box>(a, st);
        case BoxAndBall: return launch_ff<BoxAndBall>(a, st);
        case ArmWithRope: return launch_ff<ArmWithRope>(a, st);
        case Humanoid: return launch_ff<Humanoid>(a, st);
        case CpgHinge: return launch_ff<CpgHinge>(a, st);
    }
    return cudaErrorInvalidValue;
}

const char* kernel_name_fp32(int kind) {
    switch (kind) {
        case Box: return "ff_kernel<box>";
        case BoxAndBall: return "ff_kernel<box_and_ball>";
        case ArmWithRope: return "ff_kernel<arm_with_rope>";
        case Humanoid: return "ff_kernel<humanoid>";
        case CpgHinge: return "ff_kernel<cpg_hinge>";
    }
    return "?";
}

}  // namespace hb
