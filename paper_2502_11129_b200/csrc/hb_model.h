// hb_model.h — model definitions shared by the host initialiser and the
// sm_100a stepping kernels.  Compile-time topology so every kernel is fully
// specialised per ModelKind.
//
// Restates (does not include) the reference's constants and topology:
//   kSimDt / kGravity / kProjectionIterations / kBlowupLimit  simkernel.hpp:67-71
//   kStiffLink / kSoftLink                                    simkernel.cpp:13-14
//   body_count                                                simkernel.hpp:23-31
//   constraint lists (add_chain + switch)                     simkernel.cpp:35-40,95-118
//   rng::mix64 / rng::at / rng::to_unit                       rng.hpp:15-32
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define HB_HD __host__ __device__ __forceinline__
#else
#define HB_HD inline
#endif

namespace hb {

constexpr double kSimDt = 0.002;
constexpr double kGravity = 9.81;
constexpr int kIters = 8;
constexpr double kBlowupLimit = 1e6;
constexpr double kDamping = 0.8;  // build_model, simkernel.cpp:62
constexpr double kStiffLink = 2.5e5;
constexpr double kSoftLink = 1.25e5;
constexpr double kMinDist = 1e-12;  // simkernel.cpp:144

// Kinds 0-3 are hetbench::ModelKind (simkernel.hpp:14).  Kind 4 (CpgHinge)
// is NOT in the reference: the "Revolve2-style modular robot with hinge
// joints + CPG controller" of BASELINE config 3, defined in
// oracle/hb_oracle.c (its oracle) and DESIGN.md §3.6.
enum Kind : int { Box = 0, BoxAndBall = 1, ArmWithRope = 2, Humanoid = 3, CpgHinge = 4 };
constexpr int kNumKinds = 5;

HB_HD constexpr int bodies(int k) {
    return k == 0 ? 1 : k == 1 ? 2 : k == 2 ? 12 : k == 3 ? 32 : k == 4 ? 9 : 0;
}
HB_HD constexpr int constraints(int k) {
    return k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 11 : k == 3 ? 46 : k == 4 ? 12 : 0;
}
// CPG rows of kind 4: x[4], y[4], omega[4], coupling[4].
HB_HD constexpr int cpg_rows(int k) { return k == 4 ? 16 : 0; }
HB_HD constexpr int state_rows(int k) { return 6 * bodies(k) + constraints(k) + cpg_rows(k); }
// Distinct body angles build_model takes cos / sin of (simkernel.cpp:77-84:
// heading + 0.15 j per body, the humanoid's two rails share j = b % 16;
// kind 4: heading + pi/2 l per limb).  The product computes these with the
// host's libm and the rest of the initial state on the device.
HB_HD constexpr int init_angles(int k) { return k == 1 ? 2 : k == 2 ? 12 : k == 3 ? 16 : k == 4 ? 4 : 0; }

// Constraint c of model k: endpoints (a, b) and whether it is a soft link.
// Kind 4: c = 2l core-hinge (0, 1+2l), c = 2l+1 hinge-tip (1+2l, 2+2l),
// c = 8+l actuated core-tip (0, 2+2l, soft).
HB_HD constexpr int con_a(int k, int c) {
    return k == 3 ? (c < 15 ? c : c < 30 ? c + 1 : c - 30)
         : k == 4 ? (c < 8 ? (c % 2 == 0 ? 0 : c) : 0)
                  : c;
}
HB_HD constexpr int con_b(int k, int c) {
    return k == 3 ? (c < 15 ? c + 1 : c < 30 ? c + 2 : c - 30 + 16)
         : k == 4 ? (c < 8 ? c + 1 : 2 * c - 14)
                  : c + 1;
}
HB_HD constexpr bool con_soft(int k, int c) { return (k == 2 && c >= 5) || (k == 4 && c >= 8); }
HB_HD constexpr bool is_chain(int k) { return k == 1 || k == 2; }

constexpr uint64_t kCpgKey = 0xC0FFEE5EEDC0DE5Full;
constexpr double kCpgAmp = 0.2;

// ---- counter-based generator (rng.hpp:15-32) ----
HB_HD constexpr uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}
HB_HD constexpr uint64_t rng_at(uint64_t key, uint64_t ctr) {
    return mix64(mix64(key + 0x9E3779B97F4A7C15ull) ^ (ctr * 0xD1B54A32D192ED03ull + 1));
}
HB_HD constexpr double to_unit(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

// EA keys (ea.cpp:15-16)
constexpr uint64_t kInitKey = 0x8F5D4C3B2A190807ull;
constexpr uint64_t kChildKey = 0x243F6A8885A308D3ull;

// ---- FNV-1a 64 (simkernel.cpp:16-26) ----
constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
HB_HD uint64_t fnv_absorb_bits(uint64_t h, uint64_t bits) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 8; ++i) {
        h ^= (bits >> (8 * i)) & 0xffu;
        h *= kFnvPrime;
    }
    return h;
}

}  // namespace hb
