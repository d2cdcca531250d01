// ubench_fp64.cu — FP64 pipe latency / issue-rate microbenchmarks on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o ubench tools/ubench_fp64.cu
// Prints cycles per dependent op (latency) and cycles per independent op per
// warp (issue interval) for DADD, DMUL, DSETP+FSEL, FSEL, IMNMX, MUFU.RCP64H.
#include <cstdio>
#include <cstdint>

#define N_ITERS 4096

__global__ void lat_dadd(double* out, double a, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N_ITERS; ++i) x = x + a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dmul(double* out, double a, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N_ITERS; ++i) x = x * a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_sel(double* out, double a, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N_ITERS; ++i) x = (x < 0.5) ? 0.0 : x;  // DSETP + 2 FSEL
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_chain_addsel(double* out, double a, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N_ITERS; ++i) { x = x + a; x = (x < 0.0) ? 0.0 : x; }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
// throughput: 8 independent chains per thread, one warp per SMSP (block of 128)
__global__ void thr_dadd(double* out, double a, long long* cyc) {
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N_ITERS; ++i) {
        x0 = x0 + a; x1 = x1 + a; x2 = x2 + a; x3 = x3 + a;
        x4 = x4 + a; x5 = x5 + a; x6 = x6 + a; x7 = x7 + a;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void thr_dsetp(double* out, double a, long long* cyc) {
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
    bool b = false;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N_ITERS; ++i) {
        b |= fabs(x0) > 1e6; b |= fabs(x1) > 1e6; b |= fabs(x2) > 1e6; b |= fabs(x3) > 1e6;
        x0 = __longlong_as_double(__double_as_longlong(x0) ^ 1);
        x1 = __longlong_as_double(__double_as_longlong(x1) ^ 1);
        x2 = __longlong_as_double(__double_as_longlong(x2) ^ 1);
        x3 = __longlong_as_double(__double_as_longlong(x3) ^ 1);
    }
    long long t1 = clock64();
    out[threadIdx.x] = b ? x0 : x1 + x2 + x3;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_mufu(double* out, double a, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N_ITERS; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_div(double* out, double a, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_ITERS; ++i) x = 1.0000001 / x;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_sqrt(double* out, double a, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N_ITERS; ++i) x = sqrt(x) + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

// Box grounded-phase step: two independent 5-op chains (x, y) per step.
__global__ void chain_xy(double* out, double a, long long* cyc) {
    const double damp = 1.0 - 0.8 * a * 1e-3, dt = a * 2e-3, inv = 1.0 / dt;
    double px = threadIdx.x, py = 1.0, vx = 0.3, vy = -0.2;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N_ITERS; ++i) {
        const double qx = px + (vx * damp) * dt, qy = py + (vy * damp) * dt;
        vx = (qx - px) * inv; vy = (qy - py) * inv;
        px = qx; py = qy;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = px + py + vx + vy;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMallocManaged(&cyc, sizeof(long long));
    struct K { const char* name; void (*f)(double*, double, long long*); int threads; double ops; };
    K ks[] = {
        {"DADD dependent latency (cyc/op)", lat_dadd, 32, N_ITERS},
        {"DMUL dependent latency (cyc/op)", lat_dmul, 32, N_ITERS},
        {"DSETP+FSEL dependent (cyc/op)", lat_sel, 32, N_ITERS},
        {"DADD+clamp dependent (cyc/iter)", lat_chain_addsel, 32, N_ITERS},
        {"MUFU.RCP64H dependent (cyc/op)", lat_mufu, 32, N_ITERS},
        {"IEEE div dependent (cyc/op)", lat_div, 32, N_ITERS},
        {"IEEE sqrt+add dependent (cyc/op)", lat_sqrt, 32, N_ITERS},
        {"DADD 1 warp 8 chains (cyc/warp-instr)", thr_dadd, 32, 8.0 * N_ITERS},
        {"DADD 4 warps/SM 8 chains (cyc/warp-instr/SMSP)", thr_dadd, 128, 8.0 * N_ITERS},
        {"DADD 8 warps/SM 8 chains (cyc/warp-instr/SMSP)", thr_dadd, 256, 8.0 * N_ITERS / 2},
        {"DSETP 1 warp 4 chains (cyc/warp-instr)", thr_dsetp, 32, 4.0 * N_ITERS},
    };
    {
        // grounded-step chain: 1 CTA, then the full 16384-variant grid (512 x 32)
        double* big;
        cudaMalloc(&big, 16384 * sizeof(double));
        for (int grid : {1, 148, 296, 512, 592, 1184}) {
            for (int it = 0; it < 2; ++it) { chain_xy<<<grid, 32>>>(big, 1.0, cyc); cudaDeviceSynchronize(); }
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0); chain_xy<<<grid, 32>>>(big, 1.0, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("chain_xy grid %4d x 32: %6.2f cyc/step (clock64, CTA 0), %6.2f ns/step (events)\n", grid,
                   (double)*cyc / N_ITERS, ms * 1e6 / N_ITERS);
        }
    }
    for (auto& k : ks) {
        k.f<<<1, k.threads>>>(out, 1.0000001, cyc);
        cudaDeviceSynchronize();
        k.f<<<1, k.threads>>>(out, 1.0000001, cyc);
        cudaDeviceSynchronize();
        printf("%-48s %8.2f\n", k.name, (double)*cyc / k.ops);
    }
    return 0;
}
