// hb_ea.cu — device side of the (mu + lambda) generation loop
// (/root/reference/proj/src/ea.cpp:33-105).
//
//   genomes[i]   = rng::at(seed ^ kInitKey, i)                     ea.cpp:48-52
//   selection    = std::stable_sort(order, fitness[a] > fitness[b]) ea.cpp:60-72
//   offspring[i] = rng::at(parents[i] ^ kChildKey, (g << 32) + i)   ea.cpp:75-79
//   population   = parents ++ offspring                            ea.cpp:84-91
//
// Selection = the permutation std::stable_sort with `>` produces: fitness
// descending, ties in index order.  Fitness = sqrt(dx*dx + dy*dy) is +0 or a
// positive finite double for every completed variant (a blown-up variant
// aborts the generation, as batch_failure aborts run_ea), so the order of
// the IEEE bit patterns is the numeric order.  The sort runs on the high 32
// bits only (a stable radix sort of (hi32, index), at most 4 passes — half
// those of a 64-bit key), then every run of equal high words, already in index
// order, is re-sorted by (low 32 bits descending, index ascending) —
// insertion sort by the run's first thread; runs are a few elements (two
// fitness values agree in their top 32 bits ~2^-20 relative apart).
#include <atomic>
#include <cstdlib>

#include <cooperative_groups.h>
#include <cub/block/block_radix_rank.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hb_internal.h"
#include "hb_model.h"

namespace hb {

namespace {

__global__ void init_genomes_kernel(uint64_t key, size_t pop, uint64_t* genomes, uint64_t* g_dev) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < pop) genomes[i] = rng_at(key, i);
    if (g_dev && i == 0) *g_dev = 0;  // each selection's first kernel advances it (to 1 first)
}

// (high word of fitness[i], i)
__global__ void key_hi_kernel(const double* fitness, size_t n, uint32_t* key, uint32_t* idx, uint64_t* g_dev) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (g_dev && i == 0) *g_dev += 1;  // this generation's index (read by tie_select_kernel)
    if (i >= n) return;
    key[i] = static_cast<uint32_t>(__double2hiint(fitness[i]));
    idx[i] = static_cast<uint32_t>(i);
}

// Position order of two members of one run of equal high words: low word
// descending, then index ascending (a total order, so an unstable sort of
// the run gives exactly the stable sort's result).
__device__ __forceinline__ bool run_before(uint32_t ia, uint32_t ib, const double* fitness) {
    const uint32_t la = static_cast<uint32_t>(__double2loint(fitness[ia]));
    const uint32_t lb = static_cast<uint32_t>(__double2loint(fitness[ib]));
    return la > lb || (la == lb && ia < ib);
}

// Runs are a few elements, sorted by insertion; a long run (only crafted
// fitness has thousands of values sharing their top 32 bits) is heap-sorted
// instead, O(L log L) rather than O(L^2) on its one thread.
constexpr size_t kInsertionMax = 32;

__device__ void heap_sift(uint32_t* a, size_t i, size_t len, const double* fitness) {
    const uint32_t x = a[i];
    for (;;) {
        size_t c = 2 * i + 1;
        if (c >= len) break;
        if (c + 1 < len && run_before(a[c], a[c + 1], fitness)) ++c;  // the later-placed child
        if (!run_before(x, a[c], fitness)) break;
        a[i] = a[c];
        i = c;
    }
    a[i] = x;
}

__device__ void heap_sort_run(uint32_t* a, size_t len, const double* fitness) {
    for (size_t i = len / 2; i-- > 0;) heap_sift(a, i, len, fitness);
    for (size_t k = len; k-- > 1;) {
        const uint32_t t = a[0];
        a[0] = a[k];
        a[k] = t;
        heap_sift(a, 0, k, fitness);
    }
}

// Tie fix, selection and variation in one pass over the sorted order
// (ea.cpp:60-79).  The sort ordered (high word desc, index asc); within a run
// of equal high words the order must be low word descending, index
// ascending: the run's first position insertion-sorts the whole run (it may
// reach past mu) and emits, for the run's positions q < mu, parent
// next[q] = genomes[order[q]] with its fitness and offspring
// next[mu + q] = rng_at(parent ^ kChildKey, (g << 32) + q).  Runs are
// almost always of one, so each thread emits its own position (coalesced).
// g from *g_dev when given (graph replays; advanced by the sort kernel).
__global__ void tie_select_kernel(const uint64_t* genomes, const double* fitness, const uint32_t* key,
                                  size_t n, uint32_t* order, size_t mu, uint64_t g, const uint64_t* g_dev,
                                  uint64_t* next, double* next_fit) {
    const size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (p >= mu) return;
    const uint32_t kp = key[p];
    if (p > 0 && key[p - 1] == kp) return;  // inside a run: its first position emits it
    size_t end = p + 1;
    while (end < n && key[end] == kp) ++end;
    if (end - p > kInsertionMax)
        heap_sort_run(order + p, end - p, fitness);  // bounded cost for crafted long runs
    for (size_t a = p + 1; a < end && end - p <= kInsertionMax; ++a) {
        const uint32_t ia = order[a];
        const uint32_t la = static_cast<uint32_t>(__double2loint(fitness[ia]));
        size_t b = a;
        while (b > p) {
            const uint32_t ib = order[b - 1];
            const uint32_t lb = static_cast<uint32_t>(__double2loint(fitness[ib]));
            if (lb > la || (lb == la && ib < ia)) break;  // ib precedes ia
            order[b] = ib;
            --b;
        }
        order[b] = ia;
    }
    const uint64_t gen = g_dev ? *g_dev : g;
    const size_t stop = end < mu ? end : mu;
    for (size_t q = p; q < stop; ++q) {
        const uint32_t o = order[q];
        const uint64_t parent = genomes[o];
        next[q] = parent;
        next_fit[q] = fitness[o];
        next[mu + q] = rng_at(parent ^ kChildKey, (gen << 32) + q);
    }
}

__global__ void fitness_from_results_kernel(const hb_variant_result* out, size_t n, double* fitness) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) fitness[i] = out[i].fitness;
}

unsigned blocks_for(size_t n) { return static_cast<unsigned>((n + 255) / 256); }

// ---------------------------------------------------------------------------
// One-cluster radix sort of up to 65 536 (high word, index) pairs: the
// stable LSD sort of the selection in a single launch.  CTAS CTAs of THREADS
// threads form one cluster (16 x 512 where the device schedules the
// non-portable cluster, else 8 x 1 024); each holds a THREADS x ITEMS tile in
// shared memory; per 8-bit digit pass every CTA ranks its tile stably
// (cub::BlockRadixRankMatch), the CTAs exchange their digit histograms through
// distributed shared memory, and every item is scattered straight into its
// destination CTA's next tile (st.shared::cluster).  Digits no key varies in
// are skipped (a non-negative fitness of narrow exponent range: 3 passes).
// Sorting ~high word ascending = high word descending; padding
// (index >= n) gets the largest key and higher indices, so it ends up after
// every real item.  Replaces the ~20 launches of the device-wide sort (the
// passes are latency-bound at this size).  Measured and dropped: an
// mbarrier / st.async exchange with no cluster barrier inside the passes
// (1 us of 26: the passes are bound by the ranking, not the barriers).
constexpr int kSortMax = 65536;
template <int THREADS>
using SortRank = cub::BlockRadixRankMatch<THREADS, 8, false>;  // match.any ranking: small per-warp counters

template <int THREADS, int ITEMS>
struct SortSmem {
    uint2 buf[THREADS * ITEMS];  // (key, index): every CTA has read its tile into
                                 // registers before the histogram barrier, so the
                                 // scatter after it may overwrite the tile in place
    typename SortRank<THREADS>::TempStorage rank;
    int hist[256];    // this CTA's digit counts (read by the whole cluster)
    int prefix[256];  // this CTA's exclusive digit prefix
    int goff[256];    // global start of this CTA's items of each digit
    int tot[256];
    uint32_t wor[32], wand[32];  // OR / AND of each warp's keys (which digits vary at all)
    uint32_t kor, kand;          // ... of this CTA's keys
    uint32_t vary;               // the cluster's varying key bits
};

struct DigitAt {
    uint32_t shift;
    __device__ __forceinline__ uint32_t Digit(uint32_t k) const { return (k >> shift) & 0xffu; }
};

template <int CTAS, int THREADS>
__global__ void __launch_bounds__(THREADS, 1)
cluster_sort_kernel(const double* fitness, int n, uint32_t* key_out, uint32_t* idx_out, uint64_t* g_dev) {
    constexpr int ITEMS = kSortMax / (CTAS * THREADS);
    constexpr int TILE = THREADS * ITEMS;
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem<THREADS, ITEMS>& sm = *reinterpret_cast<SortSmem<THREADS, ITEMS>*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    const int t = threadIdx.x;
    if (g_dev && c == 0 && t == 0) *g_dev += 1;  // this generation's index (read by tie_select_kernel)
    // warp-striped: item j of lane l in warp w is tile position w*32*K + 32j + l —
    // the order BlockRadixRankMatch ranks ties in (warp, item, lane), so the
    // ranking is stable with respect to tile order
    const int stripe = (t >> 5) * 32 * ITEMS + (t & 31);
    uint32_t key[ITEMS], idx[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const int e = c * TILE + stripe + 32 * j;
        idx[j] = static_cast<uint32_t>(e);
        key[j] = e < n ? ~static_cast<uint32_t>(__double2hiint(fitness[e])) : 0xffffffffu;
    }
    {
        uint32_t o = 0u, a = 0xffffffffu;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (static_cast<int>(idx[j]) < n) {  // padding (all-ones keys, the highest
                o |= key[j];                     // indices) sorts last whatever digits
                a &= key[j];                     // are skipped
            }
        }
        o = __reduce_or_sync(0xffffffffu, o);
        a = __reduce_and_sync(0xffffffffu, a);
        if ((t & 31) == 0) {  // read after the barriers of the first pass
            sm.wor[t >> 5] = o;
            sm.wand[t >> 5] = a;
        }
    }
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
        // a digit no key varies in permutes nothing (the pass is the stable
        // identity): skip it — a non-negative fitness of narrow exponent range
        // leaves the top byte constant (decided from pass 0's exchange)
        if (pass > 0 && ((sm.vary >> (8 * pass)) & 0xffu) == 0u) continue;
        const uint32_t shift = 8u * pass;
        int ranks[ITEMS];
        int excl[1];
        SortRank<THREADS>(sm.rank).RankKeys(key, ranks, DigitAt{shift}, excl);
        if (t < 256) sm.prefix[t] = excl[0];
        __syncthreads();
        if (t < 256) sm.hist[t] = (t < 255 ? sm.prefix[t + 1] : TILE) - sm.prefix[t];
        if (shift == 0 && t < 32) {
            const bool w = t < THREADS / 32;
            const uint32_t o = __reduce_or_sync(0xffffffffu, w ? sm.wor[t] : 0u);
            const uint32_t a = __reduce_and_sync(0xffffffffu, w ? sm.wand[t] : 0xffffffffu);
            if (t == 0) {
                sm.kor = o;
                sm.kand = a;
            }
        }
        cluster.sync();  // every CTA's histogram (and key OR / AND) is visible
        if (shift == 0 && t == 0) {
            uint32_t o = 0u, a = 0xffffffffu;
            for (int r = 0; r < CTAS; ++r) {
                o |= *cluster.map_shared_rank(&sm.kor, r);
                a &= *cluster.map_shared_rank(&sm.kand, r);
            }
            sm.vary = o ^ a;
        }
        if (t < 256) {
            int tot = 0, before = 0;
#pragma unroll
            for (int r = 0; r < CTAS; ++r) {
                const int v = cluster.map_shared_rank(sm.hist, r)[t];
                tot += v;
                before += r < c ? v : 0;
            }
            sm.tot[t] = tot;
            sm.goff[t] = before;
        }
        __syncthreads();
        if (t < 32) {  // exclusive scan of the 256 digit totals: one warp, 8 digits per lane
            int v[8], sum = 0;
#pragma unroll
            for (int d = 0; d < 8; ++d) { v[d] = sm.tot[8 * t + d]; sum += v[d]; }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, o);
                if (t >= o) incl += u;
            }
            int run = incl - sum;
#pragma unroll
            for (int d = 0; d < 8; ++d) { sm.goff[8 * t + d] += run; run += v[d]; }
        }
        __syncthreads();
        uint2* next = sm.buf;
        const uint32_t next_sa = static_cast<uint32_t>(__cvta_generic_to_shared(next));
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t d = (key[j] >> shift) & 0xffu;
            const int pos = sm.goff[d] + ranks[j] - sm.prefix[d];
            // st.shared::cluster into the destination CTA's tile (mapa: the
            // same shared-window offset in CTA pos / tile)
            const uint32_t local = next_sa + static_cast<uint32_t>(pos % TILE) * 8u;
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(pos / TILE));
            asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" :: "r"(remote), "r"(key[j]), "r"(idx[j])
                         : "memory");
        }
        cluster.sync();  // every item has arrived in its tile
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint2 kv = next[stripe + 32 * j];
            key[j] = kv.x;
            idx[j] = kv.y;
        }
    }
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const int p = c * TILE + stripe + 32 * j;
        if (p < n) {
            key_out[p] = ~key[j];
            idx_out[p] = idx[j];
        }
    }
    cluster.sync();  // no CTA leaves while another may still read its shared memory
}

template <int CTAS, int THREADS>
cudaError_t launch_sort(const double* fitness, int n, uint32_t* key_out, uint32_t* idx_out, uint64_t* g_dev,
                        cudaStream_t st, bool probe_only = false) {
    constexpr size_t smem = sizeof(SortSmem<THREADS, kSortMax / (CTAS * THREADS)>);
    auto* kern = cluster_sort_kernel<CTAS, THREADS>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CTAS);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (probe_only) {  // opt-ins, and whether one cluster fits the device
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e == cudaSuccess && CTAS > 8)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        int clusters = 0;
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg);
        if (e == cudaSuccess && clusters < 1) e = cudaErrorInvalidConfiguration;
        return e;
    }
    return cudaLaunchKernelEx(&cfg, kern, fitness, n, key_out, idx_out, g_dev);
}

// The cluster shape, probed once per device: 16 CTAs of 512 threads
// (non-portable cluster: a quarter of the items per SM of the portable
// 8 x 1 024 and the pass time is issue-bound per SM; measured 26 vs 38 us at
// 65 536) where the device schedules it, else the portable 8 x 1 024
// (HB_SORT_CLUSTER8=1 pins it).  State: 0 = unprobed, 1 = 8 x 1 024,
// 2 = 16 x 512.
cudaError_t launch_cluster_sort(const double* fitness, int n, uint32_t* key_out, uint32_t* idx_out,
                                uint64_t* g_dev, cudaStream_t st) {
    static std::atomic<uint8_t> state[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    uint8_t s = state[dev & 63].load();
    if (s == 0) {
        if (!getenv("HB_SORT_CLUSTER8") &&
            launch_sort<16, 512>(nullptr, 0, nullptr, nullptr, nullptr, st, true) == cudaSuccess) {
            s = 2;
        } else {
            cudaGetLastError();  // a refused probe is not an error of this call
            e = launch_sort<8, 1024>(nullptr, 0, nullptr, nullptr, nullptr, st, true);
            if (e != cudaSuccess) return e;
            s = 1;
        }
        state[dev & 63].store(s);
    }
    if (s == 2) return launch_sort<16, 512>(fitness, n, key_out, idx_out, g_dev, st);
    return launch_sort<8, 1024>(fitness, n, key_out, idx_out, g_dev, st);
}

}  // namespace

cudaError_t ea_init_genomes(uint64_t seed, size_t pop, uint64_t* d_genomes, cudaStream_t st, uint64_t* g_dev) {
    if (pop == 0) return cudaSuccess;
    init_genomes_kernel<<<blocks_for(pop), 256, 0, st>>>(seed ^ kInitKey, pop, d_genomes, g_dev);
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
    cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, static_cast<const uint32_t*>(nullptr),
                                              static_cast<uint32_t*>(nullptr),
                                              static_cast<const uint32_t*>(nullptr),
                                              static_cast<uint32_t*>(nullptr), static_cast<int>(pop));
    // + keys in / out and indices in / out (pop u32 each), 256 B aligned
    auto al = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    return al(temp) + 4 * al(pop * sizeof(uint32_t));
}

namespace {

cudaError_t select_vary_impl(const uint64_t* d_genomes, const double* d_fitness, size_t pop, uint64_t g,
                             uint64_t* g_dev, uint64_t* d_next, double* d_next_fit, void* scratch,
                             size_t scratch_bytes, cudaStream_t st) {
    auto al = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, static_cast<const uint32_t*>(nullptr),
                                              static_cast<uint32_t*>(nullptr),
                                              static_cast<const uint32_t*>(nullptr),
                                              static_cast<uint32_t*>(nullptr), static_cast<int>(pop));
    const size_t words = al(pop * sizeof(uint32_t));
    if (al(temp) + 4 * words > scratch_bytes) return cudaErrorInvalidValue;
    char* base = static_cast<char*>(scratch);
    void* d_temp = base;
    uint32_t* key_in = reinterpret_cast<uint32_t*>(base + al(temp));
    uint32_t* key_out = reinterpret_cast<uint32_t*>(base + al(temp) + words);
    uint32_t* idx_in = reinterpret_cast<uint32_t*>(base + al(temp) + 2 * words);
    uint32_t* idx_out = reinterpret_cast<uint32_t*>(base + al(temp) + 3 * words);
    cudaError_t e;
    if (pop <= static_cast<size_t>(kSortMax)) {  // one cluster, one launch
        e = launch_cluster_sort(d_fitness, static_cast<int>(pop), key_out, idx_out, g_dev, st);
    } else {
        key_hi_kernel<<<blocks_for(pop), 256, 0, st>>>(d_fitness, pop, key_in, idx_in, g_dev);
        e = cub::DeviceRadixSort::SortPairsDescending(d_temp, temp, key_in, key_out, idx_in, idx_out,
                                                      static_cast<int>(pop), 0, 32, st);
    }
    if (e != cudaSuccess) return e;
    const size_t mu = pop / 2;
    tie_select_kernel<<<blocks_for(mu), 256, 0, st>>>(d_genomes, d_fitness, key_out, pop, idx_out, mu, g, g_dev,
                                                      d_next, d_next_fit);
    return cudaGetLastError();
}

}  // namespace

cudaError_t ea_select_vary(const uint64_t* d_genomes, const double* d_fitness, size_t pop, uint64_t g,
                           uint64_t* d_next, double* d_next_fit, void* scratch, size_t scratch_bytes,
                           cudaStream_t st) {
    return select_vary_impl(d_genomes, d_fitness, pop, g, nullptr, d_next, d_next_fit, scratch,
                            scratch_bytes, st);
}

// The same selection + variation captured once as a CUDA graph (the cluster
// sort + tie_select_kernel; above 65 536: key_hi + the device-wide radix
// sort's passes + tie_select_kernel) — replays pay one launch instead of one
// per kernel.  g comes from *g_dev, advanced by every replay's first kernel.
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
