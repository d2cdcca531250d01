// sort_ub.cu — CUB radix-sort cost for the EA selection (65 536 pairs):
// 64-bit keys over all bits / over the bits that vary, 32-bit keys; plain
// launches vs a captured graph.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sort_ub tools/sort_ub.cu
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <vector>
#include <random>

int main() {
    const int n = 65536;
    std::vector<double> h(n);
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> U(0.003, 1.41);
    for (auto& x : h) x = U(g);
    double *k_in, *k_out; unsigned *v_in, *v_out; void* tmp; size_t tb = 0;
    cudaMalloc(&k_in, n * 8); cudaMalloc(&k_out, n * 8); cudaMalloc(&v_in, n * 4); cudaMalloc(&v_out, n * 4);
    cudaMemcpy(k_in, h.data(), n * 8, cudaMemcpyHostToDevice);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, k_in, k_out, v_in, v_out, n);
    cudaMalloc(&tmp, tb * 2);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](int end_bit) {
        size_t t = tb * 2;
        cub::DeviceRadixSort::SortPairsDescending(tmp, t, k_in, k_out, v_in, v_out, n, 0, end_bit, st);
    };
    for (int end_bit : {64, 56}) {
        float best = 1e9;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(e0, st); run(end_bit); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        cudaGraph_t gr; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal); run(end_bit); cudaStreamEndCapture(st, &gr);
        cudaGraphInstantiate(&ge, gr, 0);
        float bestg = 1e9;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); bestg = ms < bestg ? ms : bestg;
        }
        size_t nodes = 0; cudaGraphGetNodes(gr, nullptr, &nodes);
        printf("f64 keys end_bit %d: launches %.1f us, graph %.1f us (%zu nodes)\n", end_bit, best * 1e3, bestg * 1e3, nodes);
    }
    unsigned *k32_in, *k32_out; cudaMalloc(&k32_in, n * 4); cudaMalloc(&k32_out, n * 4);
    size_t tb32 = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb32, k32_in, k32_out, v_in, v_out, n);
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
        size_t t = tb * 2;
        cudaEventRecord(e0, st);
        cub::DeviceRadixSort::SortPairsDescending(tmp, t, k32_in, k32_out, v_in, v_out, n, 0, 32, st);
        cudaEventRecord(e1, st); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("u32 keys: launches %.1f us\n", best * 1e3);
}
