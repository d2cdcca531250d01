// hb_init.cu — initial states of the multi-body models on the device
// (build_model, /root/reference/proj/src/simkernel.cpp:59-120; kind 4:
// oracle/hb_oracle.c hbo_cpg_build).
//
// Everything build_model computes is IEEE + - * and sqrt on the RngStream
// draws except cos / sin of the body angles, which must be the host libm's
// (the reference's values).  The host evaluates only those (trig rows:
// cos of angle j at row j, sin at row J + j, J = init_angles(kind)); this
// kernel repeats the rest of the construction operation for operation
// (-fmad=false, the host side is built with -ffp-contract=off) and writes
// the SoA state rows the stepping kernels read.  Against shipping the whole
// state from the host: 4 / 24 / 32 / 8 trig rows instead of 13 / 83 / 238 /
// 82 state rows over PCIe, and the host does the trig alone.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hb_internal.h"
#include "hb_model.h"

namespace hb {

namespace {

struct DevStream {  // RngStream (rng.hpp:36-49) at counter ctr
    uint64_t key, ctr;
    __device__ __forceinline__ double unit() { return to_unit(rng_at(key, ctr++)); }
    __device__ __forceinline__ double range(double lo, double hi) { return lo + (hi - lo) * unit(); }
};

template <int K>
__global__ void __launch_bounds__(128) init_kernel(const uint64_t* __restrict__ seeds,
                                                   const double* __restrict__ trig, size_t n, double* soa) {
    constexpr int nb = bodies(K);
    constexpr int m = constraints(K);
    constexpr int J = init_angles(K);
    constexpr bool twin = (K == Humanoid);
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const size_t ld = n;
    const uint64_t seed = seeds[i];
    DevStream rs{seed, 0};
    const double drop_height = rs.range(0.5, 2.0);
    const double lx = rs.range(-1.0, 1.0);
    const double ly = rs.range(-1.0, 1.0);
    rs.ctr++;  // heading: only its cos / sin are used (trig rows)
    double px[nb], py[nb], pz[nb];
#pragma unroll
    for (int b = 0; b < nb; ++b) {
        double x, y, z;
        if constexpr (K == CpgHinge) {
            if (b == 0) {
                x = 0.0;
                y = 0.0;
                z = drop_height;
            } else {
                const int l = (b - 1) / 2;
                const bool tip = ((b - 1) % 2) != 0;
                const double r = tip ? 0.50 : 0.25;
                x = r * trig[l * ld + i];
                y = r * trig[(J + l) * ld + i];
                z = drop_height + (tip ? 0.05 : 0.10);
            }
        } else {
            const double spacing = twin ? 0.12 : 0.25;
            const int j = twin ? b % 16 : b;
            const double ca = trig[j * ld + i], sa = trig[(J + j) * ld + i];
            x = spacing * static_cast<double>(j) * ca;
            y = spacing * static_cast<double>(j) * sa;
            z = drop_height + 0.05 * static_cast<double>(j);
            if (twin && b >= 16) {  // rail B offset (simkernel.cpp:85-89)
                x -= spacing * sa;
                y += spacing * ca;
            }
        }
        x += 1e-3 * rs.range(-1.0, 1.0);
        y += 1e-3 * rs.range(-1.0, 1.0);
        z += 1e-3 * rs.unit();
        px[b] = x; py[b] = y; pz[b] = z;
        soa[(3 * b + 0) * ld + i] = x;
        soa[(3 * b + 1) * ld + i] = y;
        soa[(3 * b + 2) * ld + i] = z;
        soa[(3 * nb + 3 * b + 0) * ld + i] = lx;
        soa[(3 * nb + 3 * b + 1) * ld + i] = ly;
        soa[(3 * nb + 3 * b + 2) * ld + i] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < m; ++c) {  // rest = initial distance (add_chain :35-40, rungs :112-115)
        const int A = con_a(K, c), B = con_b(K, c);
        const double dx = px[B] - px[A], dy = py[B] - py[A], dz = pz[B] - pz[A];
        soa[(6 * nb + c) * ld + i] = sqrt(dx * dx + dy * dy + dz * dz);
    }
    if constexpr (K == CpgHinge) {  // oscillator rows (hbo_cpg_build)
        DevStream cs{seed ^ kCpgKey, 0};
        double* cpg = soa + (6 * nb + m) * ld + i;
#pragma unroll
        for (int l = 0; l < 4; ++l) cpg[(8 + l) * ld] = (2.0 * 3.14159265358979323846) * cs.range(0.5, 2.0);
#pragma unroll
        for (int l = 0; l < 4; ++l) cpg[(12 + l) * ld] = cs.range(-0.5, 0.5);
#pragma unroll
        for (int l = 0; l < 4; ++l) cpg[l * ld] = cs.range(-0.1, 0.1);
#pragma unroll
        for (int l = 0; l < 4; ++l) cpg[(4 + l) * ld] = 0.0;
    }
}

}  // namespace

cudaError_t launch_init(int kind, const uint64_t* seeds, const double* trig, size_t n, double* soa,
                        cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    switch (kind) {
        case BoxAndBall: init_kernel<BoxAndBall><<<grid, 128, 0, st>>>(seeds, trig, n, soa); break;
        case ArmWithRope: init_kernel<ArmWithRope><<<grid, 128, 0, st>>>(seeds, trig, n, soa); break;
        case Humanoid: init_kernel<Humanoid><<<grid, 128, 0, st>>>(seeds, trig, n, soa); break;
        case CpgHinge: init_kernel<CpgHinge><<<grid, 128, 0, st>>>(seeds, trig, n, soa); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace hb
