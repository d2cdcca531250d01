// hb_device.cuh — device helpers shared by the FP64 stepping kernels
// (hb_kernels.cu) and the FP32 throughput mode (hb_fp32.cu): step
// coefficients, the FNV-1a absorb, the blow-up test, the CpgHinge
// oscillator and the 32-byte VariantResult epilogue.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hb_internal.h"
#include "hb_model.h"

namespace hb {
namespace {

using Coefs = StepCoefs;

__device__ __forceinline__ Coefs make_coefs(double dt) { return step_coefs(dt); }

__device__ __forceinline__ uint64_t absorb(uint64_t h, double x) {
    return fnv_absorb_bits(h, static_cast<uint64_t>(__double_as_longlong(x)));
}

__device__ __forceinline__ bool coord_ok(double x) { return fabs(x) <= kBlowupLimit; }

// CPG of the CpgHinge model (kind 4; definition in oracle/hb_oracle.c,
// hbo_cpg_step): symplectic Euler on the old state, then the actuated
// core-tip rest lengths L0 * (1 + 0.2 * clamp(x, -1, 1)).
struct Cpg {
    double x[4], y[4], w[4], c[4];
};

__device__ __forceinline__ void cpg_load(Cpg& g, const double* src, size_t ld) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        g.x[l] = __ldg(src + l * ld);
        g.y[l] = __ldg(src + (4 + l) * ld);
        g.w[l] = __ldg(src + (8 + l) * ld);
        g.c[l] = __ldg(src + (12 + l) * ld);
    }
}

__device__ __forceinline__ void cpg_update(Cpg& g, double dt, const double* l0, double* ract) {
    double nx[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) nx[l] = g.x[l] + dt * (g.w[l] * g.y[l] + g.c[l] * g.x[(l + 1) & 3]);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        g.y[l] = g.y[l] - dt * (g.w[l] * nx[l]);
        g.x[l] = nx[l];
        const double x = g.x[l];
        const double u = (x < -1.0) ? -1.0 : ((x > 1.0) ? 1.0 : x);
        ract[l] = l0[l] * (1.0 + kCpgAmp * u);
    }
}

// The 32-byte VariantResult (simkernel.hpp:51-58) of variant i; a blown-up
// variant gets {seed, 0, 0, failing step} and its step in fail[i].
__device__ __forceinline__ void emit(const SimArgs& a, size_t i, double fitness, uint64_t h,
                                     uint64_t fail) {
    const uint64_t seed = a.seeds[i];
    double2* dst = reinterpret_cast<double2*>(a.out + i);
    if (fail == 0) {
        dst[0] = make_double2(__longlong_as_double(static_cast<long long>(seed)), fitness);
        dst[1] = make_double2(__longlong_as_double(static_cast<long long>(h)),
                              __longlong_as_double(static_cast<long long>(a.steps)));
    } else {
        dst[0] = make_double2(__longlong_as_double(static_cast<long long>(seed)), 0.0);
        dst[1] = make_double2(0.0, __longlong_as_double(static_cast<long long>(fail)));
        atomicAdd(a.counters, 1u);
        if (a.fail_flag) *a.fail_flag = 1u;
    }
    a.fail[i] = fail;
}

}  // namespace
}  // namespace hb
