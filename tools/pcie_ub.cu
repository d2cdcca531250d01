// pcie_ub.cu — GPU -> mapped host memory write cost per layout (diagnostic):
// full 32-byte records (coalesced 16-byte chunks) vs only the middle 16 bytes
// of each record (fitness + checksum at offset 8) vs a contiguous 16-byte
// compact array.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pcie_ub tools/pcie_ub.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void full_rec(double2* out, size_t n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < 2 * n) out[i] = make_double2((double)i, 1.0);
}
__global__ void mid_rec(double* out, size_t n) {  // bytes 8..23 of each 32-byte record
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) { out[4 * i + 1] = (double)i; out[4 * i + 2] = 2.0; }
}
__global__ void compact(double2* out, size_t n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = make_double2((double)i, 1.0);
}

int main() {
    for (size_t n : {16384ul, 65536ul, 262144ul}) {
        void* h;
        cudaHostAlloc(&h, n * 32, cudaHostAllocMapped | cudaHostAllocPortable);
        void* d;
        cudaHostGetDevicePointer(&d, h, 0);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int k = 0; k < 3; ++k) {
            float best = 1e9;
            for (int rep = 0; rep < 20; ++rep) {
                cudaEventRecord(e0);
                if (k == 0) full_rec<<<(2 * n + 255) / 256, 256>>>((double2*)d, n);
                if (k == 1) mid_rec<<<(n + 255) / 256, 256>>>((double*)d, n);
                if (k == 2) compact<<<(n + 255) / 256, 256>>>((double2*)d, n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            const char* nm[3] = {"full 32B records", "middle 16B of 32B", "compact 16B"};
            const double bytes = k == 0 ? 32.0 * n : 16.0 * n;
            printf("n %7zu %-20s %8.2f us  %6.1f GB/s payload\n", n, nm[k], best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
        cudaFreeHost(h);
    }
}
