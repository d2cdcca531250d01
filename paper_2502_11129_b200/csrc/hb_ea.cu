// hb_ea.cu — device side of the (mu + lambda) generation loop
// (/root/reference/proj/src/ea.cpp:33-105).
//
//   genomes[i]   = rng::at(seed ^ kInitKey, i)                     ea.cpp:48-52
//   selection    = std::stable_sort(order, fitness[a] > fitness[b]) ea.cpp:60-72
//   offspring[i] = rng::at(parents[i] ^ kChildKey, (g << 32) + i)   ea.cpp:75-79
//   population   = parents ++ offspring                            ea.cpp:84-91
//
// Selection is a stable LSD radix sort of (fitness, index) pairs in
// descending key order.  Fitness = sqrt(dx*dx + dy*dy) is +0 or a positive
// finite double for every completed variant (a blown-up variant aborts the
// generation, as batch_failure aborts run_ea), so the radix order of the
// IEEE bit patterns is the numeric order and equal keys keep their input
// order — exactly the permutation std::stable_sort with `>` produces.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hb_internal.h"
#include "hb_model.h"

namespace hb {

namespace {

__global__ void init_genomes_kernel(uint64_t key, size_t pop, uint64_t* genomes) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < pop) genomes[i] = rng_at(key, i);
}

__global__ void iota_kernel(size_t n, uint32_t* idx) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) idx[i] = static_cast<uint32_t>(i);
}

// next[0, mu) = parents (genomes[order[i]]), next_fit[0, mu) = their fitness;
// next[mu + i] = offspring of parent i.
__global__ void select_vary_kernel(const uint64_t* genomes, const double* sorted_fitness,
                                   const uint32_t* order, size_t mu, uint64_t g,
                                   uint64_t* next, double* next_fit) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= mu) return;
    const uint64_t parent = genomes[order[i]];
    next[i] = parent;
    next_fit[i] = sorted_fitness[i];
    next[mu + i] = rng_at(parent ^ kChildKey, (g << 32) + i);
}

// The generation index from device memory (graph replays read the counter
// the previous replay advanced).
__global__ void select_vary_dev_g_kernel(const uint64_t* genomes, const double* sorted_fitness,
                                         const uint32_t* order, size_t mu, const uint64_t* g_dev,
                                         uint64_t* next, double* next_fit) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= mu) return;
    const uint64_t g = *g_dev;
    const uint64_t parent = genomes[order[i]];
    next[i] = parent;
    next_fit[i] = sorted_fitness[i];
    next[mu + i] = rng_at(parent ^ kChildKey, (g << 32) + i);
}

__global__ void bump_kernel(uint64_t* g_dev) { *g_dev += 1; }

__global__ void fitness_from_results_kernel(const hb_variant_result* out, size_t n, double* fitness) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) fitness[i] = out[i].fitness;
}

unsigned blocks_for(size_t n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

cudaError_t ea_init_genomes(uint64_t seed, size_t pop, uint64_t* d_genomes, cudaStream_t st) {
    if (pop == 0) return cudaSuccess;
    init_genomes_kernel<<<blocks_for(pop), 256, 0, st>>>(seed ^ kInitKey, pop, d_genomes);
    return cudaGetLastError();
}

cudaError_t ea_fitness_from_results(const hb_variant_result* out, size_t n, double* fitness,
                                    cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    fitness_from_results_kernel<<<blocks_for(n), 256, 0, st>>>(out, n, fitness);
    return cudaGetLastError();
}

size_t ea_select_scratch_bytes(size_t pop) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, static_cast<const double*>(nullptr),
                                              static_cast<double*>(nullptr),
                                              static_cast<const uint32_t*>(nullptr),
                                              static_cast<uint32_t*>(nullptr), static_cast<int>(pop));
    // + sorted keys (pop doubles) + two index arrays (pop u32 each), 256 B aligned
    auto al = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    return al(temp) + al(pop * sizeof(double)) + 2 * al(pop * sizeof(uint32_t));
}

namespace {

cudaError_t select_vary_impl(const uint64_t* d_genomes, const double* d_fitness, size_t pop, uint64_t g,
                             uint64_t* g_dev, uint64_t* d_next, double* d_next_fit, void* scratch,
                             size_t scratch_bytes, cudaStream_t st) {
    auto al = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, d_fitness, static_cast<double*>(nullptr),
                                              static_cast<const uint32_t*>(nullptr),
                                              static_cast<uint32_t*>(nullptr), static_cast<int>(pop));
    char* base = static_cast<char*>(scratch);
    void* d_temp = base;
    double* keys_out = reinterpret_cast<double*>(base + al(temp));
    uint32_t* idx_in = reinterpret_cast<uint32_t*>(base + al(temp) + al(pop * sizeof(double)));
    uint32_t* idx_out = reinterpret_cast<uint32_t*>(base + al(temp) + al(pop * sizeof(double)) +
                                                    al(pop * sizeof(uint32_t)));
    if (al(temp) + al(pop * sizeof(double)) + 2 * al(pop * sizeof(uint32_t)) > scratch_bytes)
        return cudaErrorInvalidValue;
    iota_kernel<<<blocks_for(pop), 256, 0, st>>>(pop, idx_in);
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(d_temp, temp, d_fitness, keys_out, idx_in,
                                                              idx_out, static_cast<int>(pop), 0, 64, st);
    if (e != cudaSuccess) return e;
    const size_t mu = pop / 2;
    if (g_dev) {
        select_vary_dev_g_kernel<<<blocks_for(mu), 256, 0, st>>>(d_genomes, keys_out, idx_out, mu, g_dev,
                                                                 d_next, d_next_fit);
        bump_kernel<<<1, 1, 0, st>>>(g_dev);
    } else {
        select_vary_kernel<<<blocks_for(mu), 256, 0, st>>>(d_genomes, keys_out, idx_out, mu, g, d_next,
                                                           d_next_fit);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t ea_select_vary(const uint64_t* d_genomes, const double* d_fitness, size_t pop, uint64_t g,
                           uint64_t* d_next, double* d_next_fit, void* scratch, size_t scratch_bytes,
                           cudaStream_t st) {
    return select_vary_impl(d_genomes, d_fitness, pop, g, nullptr, d_next, d_next_fit, scratch,
                            scratch_bytes, st);
}

// The same selection + variation captured once as a CUDA graph (iota, the
// radix sort's ~30 passes/launches, gather + offspring, counter bump) —
// replays pay one launch instead of one per kernel.  g comes from *g_dev,
// advanced by every replay.
cudaError_t ea_select_vary_graph(const uint64_t* d_genomes, const double* d_fitness, size_t pop,
                                 uint64_t* g_dev, uint64_t* d_next, double* d_next_fit, void* scratch,
                                 size_t scratch_bytes, cudaStream_t st, cudaGraphExec_t* exec) {
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    e = select_vary_impl(d_genomes, d_fitness, pop, 0, g_dev, d_next, d_next_fit, scratch, scratch_bytes, st);
    cudaError_t e2 = cudaStreamEndCapture(st, &graph);
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaGraphInstantiate(exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    return e;
}

}  // namespace hb
