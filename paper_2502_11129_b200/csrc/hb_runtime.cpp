// hb_runtime.cpp — host runtime behind the C ABI (include/hbgpu.h).
//
//  * host initialiser: build_model (reference src/simkernel.cpp:59-120)
//    written straight into pinned structure-of-arrays rows by a persistent
//    thread pool.  It stays on the host on purpose: glibc cos/sin are the only
//    bit-exact source of the initial arc;
//  * per-device context: stream, device + pinned buffers grown on demand;
//  * hb_run_batch = validate -> init -> H2D -> persistent kernel -> D2H,
//    the batch_executor::run contract (executor.hpp:68-73);
//  * the paper's reverse-ratio splitter, bit-for-bit (scheduler.cpp:58-87),
//    and its N-way generalisation plus a one-thread-per-device executor.
//
// Built with -O3 -ffp-contract=off (no FMA contraction: the initialiser must
// match the reference's IEEE double operation order).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvml.h>

#include "hb_internal.h"
#include "hb_model.h"

namespace {

thread_local std::string g_error;

hb_status set_global(hb_status st, const std::string& msg) {
    g_error = msg;
    return st;
}

bool valid_kind(int kind) { return kind >= 0 && kind < hb::kNumKinds; }

// ---------------------------------------------------------------------------
// Persistent fork/join pool.  The caller thread takes part; work is handed
// out in contiguous chunks (like cpu_executor, executor.cpp:93-113).  Idle
// workers spin for a short while before sleeping so that back-to-back
// batches do not pay a futex wake-up per call.
class ThreadPool {
public:
    explicit ThreadPool(int threads) : n_(std::max(1, threads)) {
        for (int t = 1; t < n_; ++t) workers_.emplace_back([this] { loop(); });
    }
    ~ThreadPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_.store(true);
            gen_.fetch_add(1);
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    int size() const { return n_; }

    // fn(begin, end) over [0, total) in contiguous chunks of at least `grain`
    // items, up to 8 per thread, taken dynamically: threads that wake late
    // (a futex wake-up after the spin window is tens of µs) find the chunks
    // already done by the caller and the early ones.
    void run(size_t total, const std::function<void(size_t, size_t)>& fn, size_t grain = 1) {
        if (total == 0) return;
        const size_t max_parts = std::max<size_t>(1, total / std::max<size_t>(1, grain));
        const int parts = n_ == 1 ? 1 : static_cast<int>(std::min<size_t>(8 * static_cast<size_t>(n_), max_parts));
        if (parts == 1) {
            fn(0, total);
            return;
        }
        Job job;
        {
            std::lock_guard<std::mutex> g(m_);
            job = Job{&fn, total, parts, ++job_id_};
            job_ = job;
            done_.store(0, std::memory_order_relaxed);
            // publishing the job id in the claim word opens the job's parts
            next_.store(job.id << 32, std::memory_order_release);
            gen_.fetch_add(1);
        }
        cv_.notify_all();
        work(job);
        while (done_.load(std::memory_order_acquire) < parts) {
        }
        std::lock_guard<std::mutex> g(m_);
        job_.fn = nullptr;
    }

private:
    // One fork/join job.  Workers copy it under the lock and claim parts
    // through `next_`, whose high 32 bits hold the job id and low 32 bits the
    // next part: a worker holding an older job's copy finds a different id
    // and claims nothing, so a late wake-up can never take (and run twice) a
    // part of the current job, and done_ counts exactly the current job's
    // parts.
    struct Job {
        const std::function<void(size_t, size_t)>* fn = nullptr;
        size_t total = 0;
        int parts = 0;
        uint64_t id = 0;
    };
    void work(const Job& job) {
        for (;;) {
            uint64_t v = next_.load(std::memory_order_acquire);
            int part;
            for (;;) {
                if ((v >> 32) != (job.id & 0xffffffffu)) return;
                part = static_cast<int>(v & 0xffffffffu);
                if (part >= job.parts) return;
                if (next_.compare_exchange_weak(v, v + 1, std::memory_order_acq_rel)) break;
            }
            const size_t chunk = job.total / job.parts, extra = job.total % job.parts;
            const size_t b = part * chunk + std::min<size_t>(part, extra);
            const size_t e = b + chunk + (static_cast<size_t>(part) < extra ? 1 : 0);
            (*job.fn)(b, e);
            done_.fetch_add(1, std::memory_order_release);
        }
    }
    void loop() {
        uint64_t seen = gen_.load();
        for (;;) {
            // spin ~100 us, then sleep on the condition variable
            auto t0 = std::chrono::steady_clock::now();
            while (gen_.load(std::memory_order_acquire) == seen) {
                if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(100)) {
                    std::unique_lock<std::mutex> lk(m_);
                    cv_.wait(lk, [&] { return gen_.load() != seen; });
                    break;
                }
            }
            seen = gen_.load();
            if (stop_.load()) return;
            Job job;
            {
                std::lock_guard<std::mutex> lk(m_);
                job = job_;
            }
            if (job.fn) work(job);
        }
    }
    int n_;
    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_;
    Job job_;               // the current job (guarded by m_)
    uint64_t job_id_ = 0;   // guarded by m_
    std::atomic<uint64_t> next_{0};
    std::atomic<int> done_{0};
    std::atomic<uint64_t> gen_{0};
    std::atomic<bool> stop_{false};
};

// One persistent host thread per device context for the multi-device calls
// (hb_run_batch_multi, the multi-context generation loop): each device gets
// its job handed over instead of a std::thread created and joined per call /
// per generation.  The worker spins briefly before sleeping, so back-to-back
// jobs (one per generation) are picked up in about a microsecond.
class DeviceWorker {
public:
    DeviceWorker() : th_([this] { loop(); }) {}
    ~DeviceWorker() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            seq_.fetch_add(1);
        }
        cv_.notify_all();
        th_.join();
    }
    void submit(std::function<void()> job) {
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = std::move(job);
            done_.store(false, std::memory_order_relaxed);
            seq_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
    }
    void wait() {
        auto t0 = std::chrono::steady_clock::now();
        while (!done_.load(std::memory_order_acquire)) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) {
                std::unique_lock<std::mutex> lk(m_);
                done_cv_.wait(lk, [&] { return done_.load(); });
                return;
            }
        }
    }

private:
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            auto t0 = std::chrono::steady_clock::now();
            while (seq_.load(std::memory_order_acquire) == seen) {
                if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) {
                    std::unique_lock<std::mutex> lk(m_);
                    cv_.wait(lk, [&] { return seq_.load() != seen; });
                    break;
                }
            }
            std::function<void()> job;
            {
                std::lock_guard<std::mutex> g(m_);
                seen = seq_.load();
                if (stop_) return;
                job = std::move(job_);
            }
            if (job) job();
            {
                std::lock_guard<std::mutex> g(m_);
                done_.store(true, std::memory_order_release);
            }
            done_cv_.notify_all();
        }
    }
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    std::function<void()> job_;
    std::atomic<uint64_t> seq_{0};
    std::atomic<bool> done_{true};
    bool stop_ = false;
    std::thread th_;
};

// ---------------------------------------------------------------------------
// NVML utilisation sampler (the accelerator side of the reference's
// UtilSampler, monitor.hpp:78-94, whose accel_percent is always 0,
// monitor.cpp:164,177).  NVML is loaded with dlopen (the driver's
// libnvidia-ml.so.1): no link-time dependency, and without NVML the trace
// holds only the final synchronised sample.  One persistent thread per
// context samples nvmlDeviceGetUtilizationRates at 20 Hz while a call is
// running.
struct Nvml {
    using init_t = nvmlReturn_t (*)();
    using by_pci_t = nvmlReturn_t (*)(const char*, nvmlDevice_t*);
    using util_t = nvmlReturn_t (*)(nvmlDevice_t, nvmlUtilization_t*);
    init_t init = nullptr;
    by_pci_t by_pci = nullptr;
    util_t util = nullptr;
    bool ok = false;
    static const Nvml& get() {
        static Nvml n = [] {
            Nvml x;
            void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
            if (!h) return x;
            x.init = reinterpret_cast<init_t>(dlsym(h, "nvmlInit_v2"));
            x.by_pci = reinterpret_cast<by_pci_t>(dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2"));
            x.util = reinterpret_cast<util_t>(dlsym(h, "nvmlDeviceGetUtilizationRates"));
            x.ok = x.init && x.by_pci && x.util && x.init() == NVML_SUCCESS;
            return x;
        }();
        return n;
    }
};

class UtilMonitor {
public:
    explicit UtilMonitor(int device) {
        const Nvml& nv = Nvml::get();
        char bus[32] = {0};
        if (nv.ok && cudaDeviceGetPCIBusId(bus, sizeof bus, device) == cudaSuccess &&
            nv.by_pci(bus, &dev_) == NVML_SUCCESS)
            have_ = true;
        cudaGetLastError();
        if (have_) th_ = std::thread([this] { loop(); });
    }
    ~UtilMonitor() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        if (th_.joinable()) th_.join();
    }
    void start() {
        std::lock_guard<std::mutex> g(m_);
        trace_.clear();
        t0_ = std::chrono::steady_clock::now();
        running_ = true;
        cv_.notify_all();
    }
    // stops sampling; appends the final synchronised sample
    std::vector<hb_util_sample> stop(double final_t, double final_percent) {
        std::unique_lock<std::mutex> lk(m_);
        running_ = false;
        trace_.push_back(hb_util_sample{final_t, final_percent});
        return trace_;
    }

private:
    void loop() {
        std::unique_lock<std::mutex> lk(m_);
        for (;;) {
            cv_.wait(lk, [&] { return stop_ || running_; });
            if (stop_) return;
            while (running_ && !stop_) {
                if (cv_.wait_for(lk, std::chrono::milliseconds(50), [&] { return stop_ || !running_; })) break;
                nvmlUtilization_t u{};
                if (Nvml::get().util(dev_, &u) == NVML_SUCCESS) {
                    const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
                    trace_.push_back(hb_util_sample{t, static_cast<double>(std::min(100u, u.gpu))});
                }
            }
        }
    }
    nvmlDevice_t dev_{};
    bool have_ = false;
    std::mutex m_;
    std::condition_variable cv_;
    bool running_ = false, stop_ = false;
    std::chrono::steady_clock::time_point t0_;
    std::vector<hb_util_sample> trace_;
    std::thread th_;
};

int default_host_threads() {
    unsigned hc = std::thread::hardware_concurrency();
    return static_cast<int>(std::min(64u, std::max(1u, hc)));
}

// ---------------------------------------------------------------------------
// build_model (simkernel.cpp:59-120) for one variant into SoA rows.
struct Stream {
    uint64_t key, ctr;
    double unit() { return hb::to_unit(hb::rng_at(key, ctr++)); }
    double range(double lo, double hi) { return lo + (hi - lo) * unit(); }  // rng.hpp:44
};

template <int K>
void build_one(uint64_t seed, double* soa, size_t ld, size_t i) {
    constexpr int n = hb::bodies(K);
    constexpr int m = hb::constraints(K);
    constexpr bool twin = (K == hb::Humanoid);
    Stream rs{seed, 0};
    const double drop_height = rs.range(0.5, 2.0);
    const double lx = rs.range(-1.0, 1.0);
    const double ly = rs.range(-1.0, 1.0);
    const double heading = rs.range(0.0, 2.0 * 3.14159265358979323846);
    const double spacing = twin ? 0.12 : 0.25;
    double px[n], py[n], pz[n];
    for (int b = 0; b < n; ++b) {
        const int j = twin ? b % 16 : b;
        const double a = heading + 0.15 * static_cast<double>(j);
        const double ca = std::cos(a), sa = std::sin(a);
        double x = spacing * static_cast<double>(j) * ca;
        double y = spacing * static_cast<double>(j) * sa;
        double z = drop_height + 0.05 * static_cast<double>(j);
        if (twin && b >= 16) {  // rail B offset (:85-89)
            x -= spacing * sa;
            y += spacing * ca;
        }
        x += 1e-3 * rs.range(-1.0, 1.0);
        y += 1e-3 * rs.range(-1.0, 1.0);
        z += 1e-3 * rs.unit();
        px[b] = x; py[b] = y; pz[b] = z;
        soa[(3 * b + 0) * ld + i] = x;
        soa[(3 * b + 1) * ld + i] = y;
        soa[(3 * b + 2) * ld + i] = z;
        soa[(3 * n + 3 * b + 0) * ld + i] = lx;
        soa[(3 * n + 3 * b + 1) * ld + i] = ly;
        soa[(3 * n + 3 * b + 2) * ld + i] = 0.0;
    }
    for (int c = 0; c < m; ++c) {  // rest = initial distance (add_chain :35-40, rungs :112-115)
        const int A = hb::con_a(K, c), B = hb::con_b(K, c);
        const double dx = px[B] - px[A], dy = py[B] - py[A], dz = pz[B] - pz[A];
        soa[(6 * n + c) * ld + i] = std::sqrt(dx * dx + dy * dy + dz * dz);
    }
}

// CpgHinge (kind 4, not in the reference; definition: oracle/hb_oracle.c
// hbo_cpg_build): core + four 2-module limbs, plus the CPG rows
// x[4], y[4], omega[4], coupling[4] after the 12 rest rows.
void build_cpg(uint64_t seed, double* soa, size_t ld, size_t i) {
    constexpr int n = 9, m = 12;
    Stream rs{seed, 0};
    const double drop_height = rs.range(0.5, 2.0);
    const double lx = rs.range(-1.0, 1.0);
    const double ly = rs.range(-1.0, 1.0);
    const double heading = rs.range(0.0, 2.0 * 3.14159265358979323846);
    double px[n], py[n], pz[n];
    for (int b = 0; b < n; ++b) {
        double x, y, z;
        if (b == 0) {
            x = 0.0; y = 0.0; z = drop_height;
        } else {
            const int l = (b - 1) / 2;
            const bool tip = ((b - 1) % 2) != 0;
            const double a = heading + 1.5707963267948966 * static_cast<double>(l);
            const double r = tip ? 0.50 : 0.25;
            x = r * std::cos(a);
            y = r * std::sin(a);
            z = drop_height + (tip ? 0.05 : 0.10);
        }
        x += 1e-3 * rs.range(-1.0, 1.0);
        y += 1e-3 * rs.range(-1.0, 1.0);
        z += 1e-3 * rs.unit();
        px[b] = x; py[b] = y; pz[b] = z;
        soa[(3 * b + 0) * ld + i] = x;
        soa[(3 * b + 1) * ld + i] = y;
        soa[(3 * b + 2) * ld + i] = z;
        soa[(3 * n + 3 * b + 0) * ld + i] = lx;
        soa[(3 * n + 3 * b + 1) * ld + i] = ly;
        soa[(3 * n + 3 * b + 2) * ld + i] = 0.0;
    }
    for (int c = 0; c < m; ++c) {
        const int A = hb::con_a(4, c), B = hb::con_b(4, c);
        const double dx = px[B] - px[A], dy = py[B] - py[A], dz = pz[B] - pz[A];
        soa[(6 * n + c) * ld + i] = std::sqrt(dx * dx + dy * dy + dz * dz);
    }
    Stream cs{seed ^ hb::kCpgKey, 0};
    double* cpg = soa + (6 * n + m) * ld + i;  // row r at cpg[r * ld]
    for (int l = 0; l < 4; ++l) cpg[(8 + l) * ld] = (2.0 * 3.14159265358979323846) * cs.range(0.5, 2.0);
    for (int l = 0; l < 4; ++l) cpg[(12 + l) * ld] = cs.range(-0.5, 0.5);
    for (int l = 0; l < 4; ++l) cpg[l * ld] = cs.range(-0.1, 0.1);
    for (int l = 0; l < 4; ++l) cpg[(4 + l) * ld] = 0.0;
}

void build_range(int kind, const uint64_t* seeds, size_t b, size_t e, double* soa, size_t ld) {
    switch (kind) {
        case 4: for (size_t i = b; i < e; ++i) build_cpg(seeds[i], soa, ld, i); break;
        case 0: for (size_t i = b; i < e; ++i) build_one<0>(seeds[i], soa, ld, i); break;
        case 1: for (size_t i = b; i < e; ++i) build_one<1>(seeds[i], soa, ld, i); break;
        case 2: for (size_t i = b; i < e; ++i) build_one<2>(seeds[i], soa, ld, i); break;
        case 3: for (size_t i = b; i < e; ++i) build_one<3>(seeds[i], soa, ld, i); break;
    }
}

// cos / sin of build_model's body angles (init_angles(kind) of them; the
// host libm's values, exactly as build_one / build_cpg take them) for the
// device initialiser: cos of angle j at row j, sin at row J + j.
void trig_range(int kind, const uint64_t* seeds, size_t b, size_t e, double* trig, size_t ld) {
    const int J = hb::init_angles(kind);
    const double step = kind == hb::CpgHinge ? 1.5707963267948966 : 0.15;
    for (size_t i = b; i < e; ++i) {
        Stream rs{seeds[i], 3};  // draw 3 = heading (after drop height, lx, ly)
        const double heading = rs.range(0.0, 2.0 * 3.14159265358979323846);
        for (int j = 0; j < J; ++j) {
            const double a = heading + step * static_cast<double>(j);
            trig[j * ld + i] = std::cos(a);
            trig[(J + j) * ld + i] = std::sin(a);
        }
    }
}

inline long long __double_as_longlong_host(double x) {
    long long v;
    std::memcpy(&v, &x, sizeof v);
    return v;
}

double elapsed_s(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// ---------------------------------------------------------------------------
struct hb_ctx {
    int device = 0;
    int sms = 148;
    int kernel_variant = HB_KERNEL_AUTO;
    int precision = HB_PRECISION_FP64;
    hb::BoxGraph box_graph;  // Box launches (optimised family, FP64)
    cudaStream_t stream = nullptr;
    std::string err;
    ThreadPool* pool = nullptr;
    DeviceWorker* worker = nullptr;  // this context's thread in multi-device calls
    int host_threads = 0;

    // device buffers
    double* d_init = nullptr;
    size_t d_init_cap = 0;  // doubles
    double* d_trig = nullptr;  // host-computed cos / sin rows for the device initialiser
    size_t d_trig_cap = 0;     // doubles
    uint64_t* d_seeds = nullptr;
    hb_variant_result* d_out = nullptr;  // 32-byte results per variant
    uint64_t* d_fail = nullptr;
    size_t d_n_cap = 0;
    unsigned* d_count = nullptr;  // failed-variant counter
    double* d_final = nullptr;
    size_t d_final_cap = 0;
    double* d_scratch = nullptr;
    double* d_ea_fit = nullptr;  // per-device fitness slice for the generation loop
    size_t d_ea_fit_cap = 0;
    // generation-loop state on the selection device, kept across hb_run_ea
    // calls (no per-call cudaMalloc / cudaFree / event creation)
    uint64_t* d_ea_gen[2] = {nullptr, nullptr};
    double* d_ea_pfit[2] = {nullptr, nullptr};
    size_t d_ea_pop_cap = 0;
    void* d_ea_scratch = nullptr;
    size_t d_ea_scratch_cap = 0;
    uint64_t* h_ea_gen = nullptr;  // pinned staging of the final population
    double* h_ea_fit = nullptr;
    cudaEvent_t ea_ev[3] = {nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> ea_timing;  // per-generation selection brackets of the queued loop
    std::vector<cudaEvent_t> ea_chain;   // multi-context loop: per-generation hand-over events
    cudaStream_t ea_copy = nullptr;      // final-population D2H overlapping the last evaluation
    cudaEvent_t ea_sel_done = nullptr;
    cudaGraphExec_t ea_graph[2] = {nullptr, nullptr};  // select/vary cur -> cur ^ 1, for d_ea_pop_cap
    size_t ea_graph_pop = 0;
    uint64_t* d_ea_g = nullptr;  // generation counter the graphs read and advance

    // pinned host buffers
    double* h_init = nullptr;
    size_t h_init_cap = 0;
    uint64_t* h_seeds = nullptr;
    hb_variant_result* h_out = nullptr;
    uint64_t* h_fail = nullptr;
    size_t h_n_cap = 0;
    unsigned* h_count = nullptr;
    unsigned* h_count_dev = nullptr;  // device address of the mapped h_count
    unsigned long long* d_ops = nullptr;  // Box executed-work counter (running total)

    // the batch currently resident on the device
    int staged_kind = -1;
    size_t staged_n = 0;
    bool staged_from_seeds = false;
    uint64_t last_steps = 0;
    uint64_t last_failed = 0;
    uint64_t last_replays = 0;
    size_t last_n = 0;
    bool counters_dirty = true;  // device counters need a reset before the next launch
    bool zero_copy = true;       // Box: read seeds / write results through host mappings
    // utilisation trace of hb_run_batch (hb_ctx_set_monitor)
    UtilMonitor* monitor = nullptr;
    cudaEvent_t mon_ev[2] = {nullptr, nullptr};  // kernel bracket of the call
    bool mon_armed = false;                       // mon_ev recorded by this call
    std::vector<hb_util_sample> util_trace;
    int fault_mode = HB_FAULT_NONE;  // hb_ctx_inject_fault (test seam)
    uint64_t fault_seed = 0;

    hb_status fail(hb_status st, const std::string& msg) {
        err = msg;
        g_error = msg;
        return st;
    }
    hb_status cuda(cudaError_t e, const char* what) {
        if (e == cudaSuccess) return HB_OK;
        return fail(HB_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    }
};

namespace {

#define HB_TRY(expr)                          \
    do {                                      \
        hb_status _st = (expr);               \
        if (_st != HB_OK) return _st;         \
    } while (0)

template <class T>
hb_status grow_dev(hb_ctx* c, T** p, size_t& cap, size_t need, const char* what) {
    if (need <= cap) return HB_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    const size_t nc = std::max(need, cap * 2);
    HB_TRY(c->cuda(cudaMalloc(reinterpret_cast<void**>(p), nc * sizeof(T)), what));
    cap = nc;
    return HB_OK;
}

hb_status ensure_capacity(hb_ctx* c, int kind, size_t n, bool need_init) {
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    if (need_init) {
        const size_t need = static_cast<size_t>(hb::state_rows(kind)) * n;
        HB_TRY(grow_dev(c, &c->d_init, c->d_init_cap, need, "cudaMalloc(init)"));
        const size_t trig = 2 * static_cast<size_t>(hb::init_angles(kind)) * n;
        if (trig) HB_TRY(grow_dev(c, &c->d_trig, c->d_trig_cap, trig, "cudaMalloc(trig)"));
        if (need > c->h_init_cap) {
            if (c->h_init) cudaFreeHost(c->h_init);
            c->h_init = nullptr;
            const size_t cap = std::max(need, c->h_init_cap * 2);
            HB_TRY(c->cuda(cudaHostAlloc(&c->h_init, cap * sizeof(double), cudaHostAllocPortable),
                           "cudaHostAlloc(init)"));
            c->h_init_cap = cap;
        }
    }
    if (n > c->d_n_cap) {
        cudaFree(c->d_seeds); cudaFree(c->d_out); cudaFree(c->d_fail);
        c->d_seeds = nullptr; c->d_out = nullptr; c->d_fail = nullptr;
        const size_t cap = std::max(n, c->d_n_cap * 2);
        HB_TRY(c->cuda(cudaMalloc(&c->d_seeds, cap * sizeof(uint64_t)), "cudaMalloc(seeds)"));
        HB_TRY(c->cuda(cudaMalloc(&c->d_out, cap * sizeof(hb_variant_result)), "cudaMalloc(out)"));
        HB_TRY(c->cuda(cudaMalloc(&c->d_fail, cap * sizeof(uint64_t)), "cudaMalloc(fail)"));
        c->d_n_cap = cap;
    }
    if (n > c->h_n_cap) {
        cudaFreeHost(c->h_seeds); cudaFreeHost(c->h_out); cudaFreeHost(c->h_fail);
        c->h_seeds = nullptr; c->h_out = nullptr; c->h_fail = nullptr;
        const size_t cap = std::max(n, c->h_n_cap * 2);
        HB_TRY(c->cuda(cudaHostAlloc(&c->h_seeds, cap * sizeof(uint64_t), cudaHostAllocPortable),
                       "cudaHostAlloc(seeds)"));
        HB_TRY(c->cuda(cudaHostAlloc(&c->h_out, cap * sizeof(hb_variant_result), 0), "cudaHostAlloc(out)"));
        HB_TRY(c->cuda(cudaHostAlloc(&c->h_fail, cap * sizeof(uint64_t), 0), "cudaHostAlloc(fail)"));
        c->h_n_cap = cap;
    }
    return HB_OK;
}

DeviceWorker& worker_of(hb_ctx* c) {
    if (!c->worker) c->worker = new DeviceWorker();
    return *c->worker;
}

ThreadPool& pool_of(hb_ctx* c) {
    if (!c->pool) c->pool = new ThreadPool(c->host_threads > 0 ? c->host_threads : default_host_threads());
    return *c->pool;
}

hb_status validate(hb_ctx* c, int kind, const void* seeds, size_t n, uint64_t steps, const void* out) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    if (!valid_kind(kind)) return c->fail(HB_INVALID_ARG, "unknown model kind " + std::to_string(kind));
    if (n == 0) return c->fail(HB_INVALID_ARG, "batch request: seeds must be non-empty");
    if (steps < 1) return c->fail(HB_INVALID_ARG, "batch request: steps must be >= 1");
    if (!seeds || !out) return c->fail(HB_INVALID_ARG, "null buffer");
    return HB_OK;
}

// Box in the optimised family builds its initial state on the device from
// the seed; every other model gets the host initialiser (glibc cos / sin).
// The FP32 throughput mode covers the multi-body models; Box keeps the FP64
// kernel in every mode (its dependent chain gains nothing from float-float
// positions: the FP32 Box loop measured 5x slower than the phase-proof one).
bool fp32_for(const hb_ctx* c, int kind) { return c->precision == HB_PRECISION_FP32 && kind != hb::Box; }

bool init_on_device(const hb_ctx* c, int kind) {
    return kind == hb::Box && c->kernel_variant == HB_KERNEL_AUTO;
}

// Multi-body kinds on the product kernels: the host computes only the libm
// cos / sin rows, the device builds the state (hb_init.cu).  The generic
// kernel variant keeps the all-host build_model (an independent path).
bool trig_init(const hb_ctx* c, int kind) {
    return kind != hb::Box && c->kernel_variant == HB_KERNEL_AUTO;
}

constexpr size_t kParallelCopyMin = 2048;  // min items per host thread for copies / assembly

// Device address of page-locked, mapped host memory (nullptr if `p` is not).
void* mapped_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost) return nullptr;
    return at.devicePointer;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

bool trace_on() {
    static int on = -1;
    if (on < 0) on = getenv("HB_TRACE") != nullptr;
    return on == 1;
}

struct Trace {
    const char* what;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    std::chrono::steady_clock::time_point last = t0;
    std::string line;
    explicit Trace(const char* w) : what(w) {}
    void mark(const char* tag) {
        if (!trace_on()) return;
        const auto now = std::chrono::steady_clock::now();
        char buf[64];
        std::snprintf(buf, sizeof buf, " %s=%.1fus", tag,
                      std::chrono::duration<double, std::micro>(now - last).count());
        line += buf;
        last = now;
    }
    ~Trace() {
        if (trace_on()) std::fprintf(stderr, "[hb] %s%s\n", what, line.c_str());
    }
};

// Seeds (+ host-built initial states) to the device.  Seeds already in
// page-locked memory are DMA'd directly; others are copied into the pinned
// staging buffer first (in parallel with the host initialiser).
hb_status stage_inputs(hb_ctx* c, int kind, const uint64_t* seeds, size_t n) {
    Trace tr("stage");
    const bool dev_init = init_on_device(c, kind);
    HB_TRY(ensure_capacity(c, kind, n, !dev_init));
    tr.mark("alloc");
    const bool direct = is_pinned(seeds);
    uint64_t* hs = c->h_seeds;
    if (dev_init) {
        if (!direct)
            pool_of(c).run(n, [&](size_t b, size_t e) {
                std::memcpy(hs + b, seeds + b, (e - b) * sizeof(uint64_t));
            }, kParallelCopyMin);
    } else if (trig_init(c, kind)) {
        double* trig = c->h_init;
        pool_of(c).run(n, [&](size_t b, size_t e) {
            if (!direct) std::memcpy(hs + b, seeds + b, (e - b) * sizeof(uint64_t));
            trig_range(kind, seeds, b, e, trig, n);
        }, 64);
        const size_t rows = 2 * static_cast<size_t>(hb::init_angles(kind));
        HB_TRY(c->cuda(cudaMemcpyAsync(c->d_trig, c->h_init, rows * n * sizeof(double),
                                       cudaMemcpyHostToDevice, c->stream), "H2D trig"));
    } else {
        double* soa = c->h_init;
        pool_of(c).run(n, [&](size_t b, size_t e) {
            if (!direct) std::memcpy(hs + b, seeds + b, (e - b) * sizeof(uint64_t));
            build_range(kind, seeds, b, e, soa, n);
        }, 64);
        const size_t rows = static_cast<size_t>(hb::state_rows(kind));
        HB_TRY(c->cuda(cudaMemcpyAsync(c->d_init, c->h_init, rows * n * sizeof(double),
                                       cudaMemcpyHostToDevice, c->stream), "H2D init"));
    }
    tr.mark(direct ? "host(direct)" : "host(staged)");
    HB_TRY(c->cuda(cudaMemcpyAsync(c->d_seeds, direct ? seeds : c->h_seeds, n * sizeof(uint64_t),
                                   cudaMemcpyHostToDevice, c->stream), "H2D seeds"));
    if (!dev_init && trig_init(c, kind))
        HB_TRY(c->cuda(hb::launch_init(kind, c->d_seeds, c->d_trig, n, c->d_init, c->stream), "init kernel"));
    tr.mark("h2d_enqueue");
    c->staged_kind = kind;
    c->staged_n = n;
    c->staged_from_seeds = dev_init;
    return HB_OK;
}

cudaError_t launch_kernel_raw(hb_ctx* c, int kind, const hb::SimArgs& a) {
    if (fp32_for(c, kind)) return hb::launch_sim_fp32(kind, a, c->stream);
    if (kind == hb::Box && c->kernel_variant == HB_KERNEL_AUTO)
        return hb::launch_box_graph(c->box_graph, a, c->stream, c->sms);
    return hb::launch_sim(kind, a, c->stream, c->sms, c->kernel_variant);
}

// One stepping launch of this context's kernel family / precision; with the
// monitor on, bracketed by CUDA events (the final utilisation sample).
cudaError_t launch_kernel(hb_ctx* c, int kind, const hb::SimArgs& a) {
    if (!c->monitor) return launch_kernel_raw(c, kind, a);
    cudaError_t e = cudaEventRecord(c->mon_ev[0], c->stream);
    if (e == cudaSuccess) e = launch_kernel_raw(c, kind, a);
    if (e == cudaSuccess) e = cudaEventRecord(c->mon_ev[1], c->stream);
    c->mon_armed = e == cudaSuccess;
    return e;
}

hb_status launch(hb_ctx* c, int kind, size_t n, uint64_t steps, double dt, bool from_seeds,
                 double* d_final) {
    if (c->counters_dirty) {
        HB_TRY(c->cuda(cudaMemsetAsync(c->d_count, 0, 2 * sizeof(unsigned), c->stream), "memset(count)"));
        c->counters_dirty = false;
    }
    hb::SimArgs a{from_seeds ? nullptr : c->d_init, c->d_seeds, n, n, steps, dt,
                  c->d_out, c->d_fail, c->d_count, d_final, nullptr, c->d_ops};
    c->last_steps = steps;
    return c->cuda(launch_kernel(c, kind, a), "kernel launch");
}

// D2H of the compact records + failure count; assemble 32-byte
// VariantResults (seed and steps are known on the host) in seed order.
// D2H of the 32-byte results (directly into `out` when it is pinned, else
// through the pinned staging buffer) + failure counters; the per-variant
// failure steps only when something blew up.
hb_status fetch(hb_ctx* c, size_t n, hb_variant_result* out, uint64_t* fail_step, bool* any_fail) {
    Trace tr("fetch");
    const bool direct = is_pinned(out);
    HB_TRY(c->cuda(cudaMemcpyAsync(direct ? out : c->h_out, c->d_out, n * sizeof(hb_variant_result),
                                   cudaMemcpyDeviceToHost, c->stream), "D2H results"));
    HB_TRY(c->cuda(cudaMemcpyAsync(c->h_count, c->d_count, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                                   c->stream), "D2H count"));
    tr.mark(direct ? "enqueue(direct)" : "enqueue(staged)");
    HB_TRY(c->cuda(cudaStreamSynchronize(c->stream), "stream sync"));
    tr.mark("sync");
    const bool any = c->h_count[0] != 0;
    c->last_failed = c->h_count[0];
    c->last_replays = c->h_count[1];
    c->last_n = n;
    // Reset the counters now (stream-ordered), so the next launch needs no
    // extra operation on its critical path.
    c->counters_dirty = (c->h_count[0] | c->h_count[1]) != 0;
    if (any || fail_step) {
        if (any) {
            HB_TRY(c->cuda(cudaMemcpy(c->h_fail, c->d_fail, n * sizeof(uint64_t), cudaMemcpyDeviceToHost),
                           "D2H fail"));
        }
    }
    const hb_variant_result* src = c->h_out;
    const uint64_t* hf = c->h_fail;
    if (!direct || fail_step) {
        pool_of(c).run(n, [&](size_t b, size_t e) {
            if (!direct) std::memcpy(out + b, src + b, (e - b) * sizeof(hb_variant_result));
            if (fail_step) {
                if (any) std::memcpy(fail_step + b, hf + b, (e - b) * sizeof(uint64_t));
                else std::memset(fail_step + b, 0, (e - b) * sizeof(uint64_t));
            }
        }, kParallelCopyMin);
    }
    tr.mark("host");
    *any_fail = any;
    return HB_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

int hb_abi_version(void) { return HBGPU_ABI_VERSION; }

int hb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int hb_body_count(int kind) { return valid_kind(kind) ? hb::bodies(kind) : -1; }
int hb_constraint_count(int kind) { return valid_kind(kind) ? hb::constraints(kind) : -1; }
int hb_state_rows(int kind) { return valid_kind(kind) ? hb::state_rows(kind) : -1; }
const char* hb_global_error(void) { return g_error.c_str(); }

hb_status hb_ctx_create(int device, hb_ctx** out) {
    if (!out) return set_global(HB_INVALID_ARG, "null output pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return set_global(HB_NO_DEVICE, std::string("no CUDA device: ") +
                                            (e != cudaSuccess ? cudaGetErrorString(e) : "count = 0"));
    }
    if (device < 0 || device >= count)
        return set_global(HB_INVALID_ARG, "device ordinal out of range");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
        return set_global(HB_NO_DEVICE, "cudaGetDeviceProperties failed");
    // The library carries sm_100a code only (no PTX): arch-specific code loads
    // on compute capability 10.0 alone, so anything else (e.g. sm_103) would
    // create a context whose every launch fails with no-kernel-image.
    if (prop.major != 10 || prop.minor != 0)
        return set_global(HB_NO_DEVICE, "device is sm_" + std::to_string(prop.major) +
                                            std::to_string(prop.minor) +
                                            "; this build targets sm_100a only");
    hb_ctx* c = new hb_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&c->d_scratch, 64) != cudaSuccess ||
        cudaMalloc(&c->d_count, 16) != cudaSuccess ||
        cudaMalloc(&c->d_ops, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(c->d_ops, 0, sizeof(unsigned long long)) != cudaSuccess ||
        cudaHostAlloc(&c->h_count, 16, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
        delete c;
        return set_global(HB_CUDA_ERROR, "stream/scratch creation failed");
    }
    c->h_count_dev = static_cast<unsigned*>(mapped_device_ptr(c->h_count));
    if (!c->h_count_dev) {
        hb_ctx_destroy(c);
        return set_global(HB_CUDA_ERROR, "mapped counter has no device address");
    }
    *out = c;
    return HB_OK;
}

void hb_ctx_destroy(hb_ctx* c) {
    if (!c) return;
    delete c->worker;
    delete c->monitor;
    for (cudaEvent_t e : c->mon_ev) if (e) cudaEventDestroy(e);
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    cudaFree(c->d_init); cudaFree(c->d_trig); cudaFree(c->d_seeds); cudaFree(c->d_out); cudaFree(c->d_fail);
    cudaFree(c->d_final); cudaFree(c->d_scratch); cudaFree(c->d_count); cudaFree(c->d_ea_fit);
    cudaFree(c->d_ops);
    hb::destroy_box_graph(c->box_graph);
    for (int k = 0; k < 2; ++k) { cudaFree(c->d_ea_gen[k]); cudaFree(c->d_ea_pfit[k]); }
    cudaFree(c->d_ea_scratch);
    cudaFreeHost(c->h_ea_gen); cudaFreeHost(c->h_ea_fit);
    for (cudaEvent_t e : c->ea_ev) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ea_timing) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ea_chain) cudaEventDestroy(e);
    if (c->ea_sel_done) cudaEventDestroy(c->ea_sel_done);
    if (c->ea_copy) cudaStreamDestroy(c->ea_copy);
    for (cudaGraphExec_t g : c->ea_graph) if (g) cudaGraphExecDestroy(g);
    cudaFree(c->d_ea_g);
    cudaFreeHost(c->h_init); cudaFreeHost(c->h_seeds); cudaFreeHost(c->h_out); cudaFreeHost(c->h_fail);
    cudaFreeHost(c->h_count);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c->pool;
    delete c;
}

const char* hb_last_error(const hb_ctx* c) { return c ? c->err.c_str() : g_error.c_str(); }
int hb_ctx_device(const hb_ctx* c) { return c ? c->device : -1; }
void* hb_ctx_stream(hb_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

hb_status hb_ctx_set_host_threads(hb_ctx* c, int threads) {
    if (!c || threads < 0) return set_global(HB_INVALID_ARG, "bad arguments");
    delete c->pool;
    c->pool = nullptr;
    c->host_threads = threads;
    return HB_OK;
}

void* hb_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (bytes == 0 ||
        cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError();
        set_global(HB_CUDA_ERROR, "cudaHostAlloc failed");
        return nullptr;
    }
    return p;
}

void hb_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

hb_status hb_last_fail_steps(hb_ctx* c, uint64_t* fail_step, size_t n) {
    if (!c || !fail_step) return set_global(HB_INVALID_ARG, "bad arguments");
    if (n > c->last_n) return c->fail(HB_INVALID_ARG, "more failure steps requested than the batch had");
    if (c->last_failed) std::memcpy(fail_step, c->h_fail, n * sizeof(uint64_t));
    else std::memset(fail_step, 0, n * sizeof(uint64_t));
    return HB_OK;
}

hb_status hb_work_counter(hb_ctx* c, uint64_t* ops) {
    if (!c || !ops) return set_global(HB_INVALID_ARG, "bad arguments");
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    HB_TRY(c->cuda(cudaStreamSynchronize(c->stream), "stream sync"));
    unsigned long long v = 0;
    HB_TRY(c->cuda(cudaMemcpy(&v, c->d_ops, sizeof v, cudaMemcpyDeviceToHost), "D2H ops"));
    *ops = v;
    return HB_OK;
}

hb_status hb_last_launch_stats(hb_ctx* c, uint64_t* failed, uint64_t* exact_replays) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    if (failed) *failed = c->last_failed;
    if (exact_replays) *exact_replays = c->last_replays;
    return HB_OK;
}

hb_status hb_ctx_set_zero_copy(hb_ctx* c, int enable) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    c->zero_copy = enable != 0;
    return HB_OK;
}

hb_status hb_ctx_set_precision(hb_ctx* c, int precision) {
    if (!c || (precision != HB_PRECISION_FP64 && precision != HB_PRECISION_FP32))
        return set_global(HB_INVALID_ARG, "bad precision");
    c->precision = precision;
    c->staged_kind = -1;
    return HB_OK;
}

hb_status hb_ctx_set_kernel(hb_ctx* c, int variant) {
    if (!c || (variant != HB_KERNEL_AUTO && variant != HB_KERNEL_GENERIC))
        return set_global(HB_INVALID_ARG, "bad kernel variant");
    c->kernel_variant = variant;
    c->staged_kind = -1;
    return HB_OK;
}

hb_status hb_build_states(int kind, const uint64_t* seeds, size_t n, double* soa, size_t ld) {
    if (!valid_kind(kind)) return set_global(HB_INVALID_ARG, "unknown model kind");
    if (!seeds || !soa || ld < n) return set_global(HB_INVALID_ARG, "bad buffers");
    build_range(kind, seeds, 0, n, soa, ld);
    return HB_OK;
}

// Box with seeds and results both in mapped page-locked memory: the kernel
// reads the seeds and writes the 32-byte results through the host mapping
// (zero-copy) — no H2D / D2H operations on the call's critical path; a
// host-mapped flag tells whether anything blew up.
static hb_status run_box_zero_copy(hb_ctx* c, const uint64_t* dseeds, hb_variant_result* dout, size_t n,
                                   uint64_t steps, uint64_t* fail_step, bool* any) {
    Trace tr("zero-copy");
    HB_TRY(ensure_capacity(c, hb::Box, n, false));
    tr.mark("capacity");
    if (c->counters_dirty) {
        HB_TRY(c->cuda(cudaMemsetAsync(c->d_count, 0, 2 * sizeof(unsigned), c->stream), "memset(count)"));
        c->counters_dirty = false;
    }
    volatile unsigned* flag = reinterpret_cast<volatile unsigned*>(c->h_count + 2);
    *flag = 0u;
    unsigned* dflag = c->h_count_dev;
    hb::SimArgs a{nullptr, dseeds, n, n, steps, hb::kSimDt, dout, c->d_fail, c->d_count, nullptr,
                  reinterpret_cast<volatile unsigned*>(dflag + 2), c->d_ops};
    c->staged_kind = -1;
    tr.mark("args");
    HB_TRY(c->cuda(launch_kernel(c, hb::Box, a), "kernel launch"));
    tr.mark("launch");
    HB_TRY(c->cuda(cudaStreamSynchronize(c->stream), "stream sync"));
    tr.mark("sync");
    c->last_n = n;
    c->last_replays = 0;
    *any = *flag != 0u;
    if (*any) {
        HB_TRY(c->cuda(cudaMemcpy(c->h_fail, c->d_fail, n * sizeof(uint64_t), cudaMemcpyDeviceToHost),
                       "D2H fail"));
        c->last_failed = 0;
        for (size_t i = 0; i < n; ++i) c->last_failed += c->h_fail[i] != 0;
        c->counters_dirty = true;
    } else {
        c->last_failed = 0;
    }
    if (fail_step) {
        if (*any) std::memcpy(fail_step, c->h_fail, n * sizeof(uint64_t));
        else std::memset(fail_step, 0, n * sizeof(uint64_t));
    }
    return HB_OK;
}

// HB_FAULT_BLOWUP: the injected variants' records become blow-ups at step 1
// (host side, after the real batch; the failure steps of the batch are kept
// in h_fail for hb_last_fail_steps).
static void apply_blowup_fault(hb_ctx* c, const uint64_t* seeds, size_t n, hb_variant_result* out,
                               uint64_t* fail_step, bool* any) {
    if (c->fault_mode != HB_FAULT_BLOWUP) return;
    bool hit = false;
    for (size_t i = 0; i < n && !hit; ++i) hit = seeds[i] == c->fault_seed;
    if (!hit) return;
    if (!*any) std::memset(c->h_fail, 0, n * sizeof(uint64_t));
    for (size_t i = 0; i < n; ++i) {
        if (seeds[i] != c->fault_seed) continue;
        if (c->h_fail[i] == 0) ++c->last_failed;
        out[i] = hb_variant_result{seeds[i], 0.0, 0, 1};
        c->h_fail[i] = 1;
        if (fail_step) fail_step[i] = 1;
    }
    *any = true;
}

static hb_status run_batch_impl(hb_ctx* c, int kind, const uint64_t* seeds, size_t n, uint64_t steps,
                                hb_variant_result* out, uint64_t* fail_step, double* wall_time_s,
                                std::chrono::steady_clock::time_point t0);

// The drop-in call.  With the monitor on (hb_ctx_set_monitor) the call is
// sampled by the context's NVML thread and closed by one synchronised
// sample: the share of the call's wall time the stepping kernel ran
// (CUDA events around the launch) — NVML's "percent of time a kernel was
// executing", exact for this call.
hb_status hb_run_batch(hb_ctx* c, int kind, const uint64_t* seeds, size_t n, uint64_t steps,
                       hb_variant_result* out, uint64_t* fail_step, double* wall_time_s) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!c || !c->monitor) return run_batch_impl(c, kind, seeds, n, steps, out, fail_step, wall_time_s, t0);
    c->monitor->start();
    c->mon_armed = false;
    double wall = 0.0;
    const hb_status st = run_batch_impl(c, kind, seeds, n, steps, out, fail_step, &wall, t0);
    if (wall_time_s) *wall_time_s = wall;
    double busy = 0.0;
    float ms = 0.f;
    if (c->mon_armed && cudaEventSynchronize(c->mon_ev[1]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, c->mon_ev[0], c->mon_ev[1]) == cudaSuccess && wall > 0.0)
        busy = std::min(100.0, 100.0 * 1e-3 * ms / wall);
    cudaGetLastError();
    c->util_trace = c->monitor->stop(wall, busy);
    return st;
}

static hb_status run_batch_impl(hb_ctx* c, int kind, const uint64_t* seeds, size_t n, uint64_t steps,
                                hb_variant_result* out, uint64_t* fail_step, double* wall_time_s,
                                std::chrono::steady_clock::time_point t0) {
    HB_TRY(validate(c, kind, seeds, n, steps, out));
    if (c->fault_mode == HB_FAULT_DEVICE)
        return c->fail(HB_CUDA_ERROR, "injected device fault (hb_ctx_inject_fault)");
    if (kind == hb::Box && c->kernel_variant == HB_KERNEL_AUTO && c->zero_copy) {
        Trace tr("ptrs");
        void* ds = mapped_device_ptr(seeds);
        void* dout = mapped_device_ptr(out);
        tr.mark("lookup");
        if (ds && dout) {
            bool any = false;
            HB_TRY(run_box_zero_copy(c, static_cast<const uint64_t*>(ds),
                                     static_cast<hb_variant_result*>(dout), n, steps, fail_step, &any));
            apply_blowup_fault(c, seeds, n, out, fail_step, &any);
            if (wall_time_s) *wall_time_s = std::max(elapsed_s(t0), 1e-9);
            if (any) return c->fail(HB_BLOWUP_PARTIAL, "numerical blow-up in batch");
            return HB_OK;
        }
    }
    HB_TRY(stage_inputs(c, kind, seeds, n));
    HB_TRY(launch(c, kind, n, steps, hb::kSimDt, c->staged_from_seeds, nullptr));
    bool any = false;
    HB_TRY(fetch(c, n, out, fail_step, &any));
    apply_blowup_fault(c, seeds, n, out, fail_step, &any);
    if (wall_time_s) *wall_time_s = std::max(elapsed_s(t0), 1e-9);
    if (any) return c->fail(HB_BLOWUP_PARTIAL, "numerical blow-up in batch");
    return HB_OK;
}

hb_status hb_ctx_reserve(hb_ctx* c, int kind, size_t n) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    if (n == 0) return HB_OK;
    std::vector<uint64_t> seeds(n);
    for (size_t i = 0; i < n; ++i) seeds[i] = i;
    std::vector<hb_variant_result> out(n);
    const hb_status st =
        run_batch_impl(c, kind, seeds.data(), n, 1, out.data(), nullptr, nullptr, std::chrono::steady_clock::now());
    return st == HB_BLOWUP_PARTIAL ? HB_OK : st;
}

hb_status hb_ctx_set_monitor(hb_ctx* c, int enable) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    if (!enable) {
        delete c->monitor;
        c->monitor = nullptr;
        c->util_trace.clear();
        return HB_OK;
    }
    if (c->monitor) return HB_OK;
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    for (cudaEvent_t& e : c->mon_ev)
        if (!e) HB_TRY(c->cuda(cudaEventCreate(&e), "event"));
    c->monitor = new UtilMonitor(c->device);
    return HB_OK;
}

hb_status hb_last_utilization(const hb_ctx* c, hb_util_sample* out, size_t cap, size_t* count) {
    if (!c || !count) return set_global(HB_INVALID_ARG, "bad arguments");
    *count = c->util_trace.size();
    if (out)
        for (size_t i = 0; i < std::min(cap, c->util_trace.size()); ++i) out[i] = c->util_trace[i];
    return HB_OK;
}

hb_status hb_ctx_inject_fault(hb_ctx* c, int mode, uint64_t seed) {
    if (!c || mode < HB_FAULT_NONE || mode > HB_FAULT_DEVICE) return set_global(HB_INVALID_ARG, "bad arguments");
    c->fault_mode = mode;
    c->fault_seed = seed;
    return HB_OK;
}

hb_status hb_run_states(hb_ctx* c, int kind, const double* init_soa, size_t n, uint64_t steps,
                        double dt, const uint64_t* seeds, hb_variant_result* out,
                        uint64_t* fail_step, double* final_soa) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    if (!valid_kind(kind)) return c->fail(HB_INVALID_ARG, "unknown model kind");
    if (!init_soa || !out || n == 0) return c->fail(HB_INVALID_ARG, "bad buffers");
    if (steps < 1) return c->fail(HB_INVALID_ARG, "simulate: steps must be >= 1");
    if (!(dt > 0.0)) return c->fail(HB_INVALID_ARG, "step: dt must be > 0");
    HB_TRY(ensure_capacity(c, kind, n, true));
    const size_t rows = static_cast<size_t>(hb::state_rows(kind));
    const size_t bytes = rows * n * sizeof(double);
    if (final_soa) HB_TRY(grow_dev(c, &c->d_final, c->d_final_cap, rows * n, "cudaMalloc(final)"));
    HB_TRY(c->cuda(cudaMemcpyAsync(c->d_init, init_soa, bytes, cudaMemcpyHostToDevice, c->stream), "H2D"));
    std::vector<uint64_t> zeros;
    const uint64_t* sd = seeds;
    if (!sd) {
        zeros.assign(n, 0);
        sd = zeros.data();
    }
    HB_TRY(c->cuda(cudaMemcpyAsync(c->d_seeds, sd, n * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                   c->stream), "H2D seeds"));
    c->staged_kind = -1;
    HB_TRY(launch(c, kind, n, steps, dt, false, final_soa ? c->d_final : nullptr));
    bool any = false;
    HB_TRY(fetch(c, n, out, fail_step, &any));
    if (final_soa) {
        HB_TRY(c->cuda(cudaMemcpy(final_soa, c->d_final, bytes, cudaMemcpyDeviceToHost), "D2H final"));
    }
    if (any) return c->fail(HB_BLOWUP_PARTIAL, "numerical blow-up in batch");
    return HB_OK;
}

hb_status hb_stage(hb_ctx* c, int kind, const uint64_t* seeds, size_t n) {
    HB_TRY(validate(c, kind, seeds, n, 1, seeds));
    HB_TRY(stage_inputs(c, kind, seeds, n));
    return c->cuda(cudaStreamSynchronize(c->stream), "stream sync");
}

hb_status hb_launch(hb_ctx* c, uint64_t steps) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    if (c->staged_kind < 0) return c->fail(HB_INVALID_ARG, "hb_launch: no staged batch");
    if (steps < 1) return c->fail(HB_INVALID_ARG, "batch request: steps must be >= 1");
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    return launch(c, c->staged_kind, c->staged_n, steps, hb::kSimDt, c->staged_from_seeds, nullptr);
}

hb_status hb_synchronize(hb_ctx* c) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    return c->cuda(cudaStreamSynchronize(c->stream), "stream sync");
}

hb_status hb_fetch(hb_ctx* c, hb_variant_result* out, uint64_t* fail_step) {
    if (!c || !out) return set_global(HB_INVALID_ARG, "bad arguments");
    if (c->staged_kind < 0) return c->fail(HB_INVALID_ARG, "hb_fetch: no staged batch");
    bool any = false;
    HB_TRY(fetch(c, c->staged_n, out, fail_step, &any));
    if (any) return c->fail(HB_BLOWUP_PARTIAL, "numerical blow-up in batch");
    return HB_OK;
}

hb_status hb_kernel_name(int kind, size_t n, char* buf, size_t cap) {
    if (!valid_kind(kind) || !buf || cap == 0) return set_global(HB_INVALID_ARG, "bad arguments");
    std::snprintf(buf, cap, "%s", hb::kernel_name(kind, n, HB_KERNEL_AUTO));
    return HB_OK;
}

int hb_format_blowup(uint64_t seed, uint64_t fail_step, double dt, char* buf, size_t cap) {
    double t = 0.0;
    for (uint64_t s = 0; s < fail_step; ++s) t += dt;  // WorldState::time += dt (:163)
    const std::string msg = "coordinate left the stable regime at t=" + std::to_string(t) +
                            " (seed " + std::to_string(seed) + ")";
    if (buf && cap) std::snprintf(buf, cap, "%s", msg.c_str());
    return static_cast<int>(msg.size());
}

// plan_allocation — scheduler.cpp:58-87, bit-for-bit.
hb_status hb_plan_allocation(double t_cpu, double t_accel, int cpu_ok, int accel_ok,
                             uint64_t n_total, hb_allocation_plan* out) {
    if (!out) return set_global(HB_INVALID_ARG, "null plan");
    if (n_total < 1) return set_global(HB_INVALID_ARG, "plan_allocation: n_total must be >= 1");
    hb_allocation_plan p{};
    p.n_total = n_total;
    if (!accel_ok) {
        p.n_accel = 0;
    } else if (!cpu_ok) {
        p.n_accel = n_total;
        p.requested_accel_fraction = 1.0;
    } else {
        const double f = t_cpu / (t_cpu + t_accel);
        p.requested_accel_fraction = f;
        uint64_t na = static_cast<uint64_t>(std::llround(f * static_cast<double>(n_total)));
        na = std::min(na, n_total);
        const double thr = 1.0 / (2.0 * static_cast<double>(n_total));
        if (na == 0 && f >= thr) na = 1;
        if (na == n_total && (1.0 - f) >= thr) na = n_total - 1;
        p.n_accel = na;
    }
    p.n_cpu = n_total - p.n_accel;
    p.accel_fraction = static_cast<double>(p.n_accel) / static_cast<double>(n_total);
    *out = p;
    return HB_OK;
}

hb_status hb_plan_allocation_n(const double* t_s, const int* ok, int count, uint64_t n_total,
                               uint64_t* shares) {
    if (!t_s || !shares || count < 1) return set_global(HB_INVALID_ARG, "bad arguments");
    if (n_total < 1) return set_global(HB_INVALID_ARG, "plan_allocation: n_total must be >= 1");
    int alive = 0;
    for (int d = 0; d < count; ++d) alive += (!ok || ok[d]) ? 1 : 0;
    if (alive == 0) return set_global(HB_INVALID_ARG, "calibrate: all back-ends failed");
    uint64_t remaining = n_total;
    for (int d = count - 1; d >= 1; --d) {
        const bool ok_d = !ok || ok[d];
        // Aggregate of devices 0..d-1 (the "cpu" side of the 2-way plan).
        bool rest_ok = false;
        double inv_sum = 0.0;
        int rest_alive = 0;
        for (int j = 0; j < d; ++j)
            if (!ok || ok[j]) {
                rest_ok = true;
                inv_sum += 1.0 / t_s[j];
                ++rest_alive;
            }
        double t_rest = 0.0;
        if (rest_alive == 1) {
            for (int j = 0; j < d; ++j)
                if (!ok || ok[j]) t_rest = t_s[j];
        } else if (rest_alive > 1) {
            t_rest = 1.0 / inv_sum;
        }
        if (remaining == 0) {
            shares[d] = 0;
            continue;
        }
        hb_allocation_plan p;
        hb_plan_allocation(t_rest, t_s[d], rest_ok ? 1 : 0, ok_d ? 1 : 0, remaining, &p);
        shares[d] = p.n_accel;
        remaining -= p.n_accel;
    }
    shares[0] = remaining;
    return HB_OK;
}

// N-way run_hybrid (scheduler.cpp:113-211) over device contexts: contiguous
// slices in device order, one persistent worker thread per device, merged in
// seed order.  A device that fails its slice with anything but a blow-up
// (HB_BLOWUP_PARTIAL is the batch's own result: re-running it elsewhere
// reproduces it) is dead for the rest of the call, and its slice is
// re-planned over the surviving devices by hb_plan_allocation_n (ok = 0 for
// the dead), in proportion to the shares the survivors were given — the N-way
// form of the reference's re-dispatch (:162-183); the result is degraded.
hb_status hb_run_batch_multi(hb_ctx* const* ctxs, int count, const uint64_t* shares, int kind,
                             const uint64_t* seeds, size_t n, uint64_t steps,
                             hb_variant_result* out, uint64_t* fail_step,
                             double* per_device_wall_s, double* wall_time_s,
                             int* device_ok, int* degraded) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!ctxs || count < 1) return set_global(HB_INVALID_ARG, "no contexts");
    for (int d = 0; d < count; ++d)
        if (!ctxs[d]) return set_global(HB_INVALID_ARG, "null context");
    if (!valid_kind(kind)) return set_global(HB_INVALID_ARG, "unknown model kind");
    if (n == 0) return set_global(HB_INVALID_ARG, "batch request: seeds must be non-empty");
    if (steps < 1) return set_global(HB_INVALID_ARG, "batch request: steps must be >= 1");
    if (!seeds || !out) return set_global(HB_INVALID_ARG, "null buffer");
    std::vector<uint64_t> sh(count);
    if (shares) {
        uint64_t sum = 0;
        for (int d = 0; d < count; ++d) sum += (sh[d] = shares[d]);
        if (sum != n) return set_global(HB_INVALID_ARG, "shares do not sum to the batch size");
    } else {
        for (int d = 0; d < count; ++d) sh[d] = n / count + (static_cast<uint64_t>(d) < n % count ? 1 : 0);
    }
    // re-dispatch weights: a device's original share is its throughput
    std::vector<double> weight(count);
    for (int d = 0; d < count; ++d) weight[d] = sh[d] > 0 ? 1.0 / static_cast<double>(sh[d]) : 1.0;
    std::vector<int> alive(count, 1);
    std::vector<double> walls(count, 0.0);
    std::vector<hb_status> st(count, HB_OK);
    std::vector<std::string> err(count);
    struct Slice { size_t b, len; };
    std::vector<std::vector<Slice>> work(count);
    {
        size_t begin = 0;
        for (int d = 0; d < count; ++d) {
            if (sh[d]) work[d].push_back({begin, sh[d]});
            begin += sh[d];
        }
    }
    bool blow = false, lost = false;
    std::string first_err;
    hb_status first_st = HB_OK;
    for (;;) {
        std::vector<int> busy;
        for (int d = 0; d < count; ++d) {
            if (work[d].empty()) continue;
            busy.push_back(d);
            worker_of(ctxs[d]).submit([&, d] {
                st[d] = HB_OK;
                for (const Slice& s : work[d]) {
                    double w = 0.0;
                    const hb_status r = hb_run_batch(ctxs[d], kind, seeds + s.b, s.len, steps, out + s.b,
                                                     fail_step ? fail_step + s.b : nullptr, &w);
                    walls[d] += w;
                    if (r == HB_BLOWUP_PARTIAL) {
                        if (st[d] == HB_OK) st[d] = r;
                    } else if (r != HB_OK) {
                        st[d] = r;
                        err[d] = hb_last_error(ctxs[d]);
                        return;
                    }
                }
            });
        }
        if (busy.empty()) break;
        for (int d : busy) worker_of(ctxs[d]).wait();
        std::vector<Slice> orphans;
        for (int d : busy) {
            if (st[d] == HB_BLOWUP_PARTIAL) blow = true;
            if (st[d] == HB_OK || st[d] == HB_BLOWUP_PARTIAL) {
                work[d].clear();
                continue;
            }
            if (first_st == HB_OK) {
                first_st = st[d];
                first_err = "device " + std::to_string(d) + ": " + err[d];
            }
            alive[d] = 0;
            lost = true;
            orphans.insert(orphans.end(), work[d].begin(), work[d].end());
            work[d].clear();
        }
        if (orphans.empty()) break;
        if (std::find(alive.begin(), alive.end(), 1) == alive.end()) {
            if (device_ok) for (int d = 0; d < count; ++d) device_ok[d] = 0;
            return set_global(first_st, "all devices failed; " + first_err);
        }
        for (const Slice& o : orphans) {
            std::vector<uint64_t> part(count);
            hb_plan_allocation_n(weight.data(), alive.data(), count, o.len, part.data());
            size_t b = o.b;
            for (int d = 0; d < count; ++d) {
                if (part[d]) work[d].push_back({b, part[d]});
                b += part[d];
            }
        }
    }
    if (per_device_wall_s)
        for (int d = 0; d < count; ++d) per_device_wall_s[d] = walls[d];
    if (device_ok)
        for (int d = 0; d < count; ++d) device_ok[d] = alive[d];
    if (degraded) *degraded = lost ? 1 : 0;
    if (wall_time_s) *wall_time_s = std::max(elapsed_s(t0), 1e-9);
    if (blow) return set_global(HB_BLOWUP_PARTIAL, "numerical blow-up in batch");
    return HB_OK;
}

// Probe timing on one context (hb_calibrate): stage seeds 0..probe_n-1 once,
// then `repeats` samples of back-to-back launches bracketed by CUDA events on
// the context's stream, each sample >= 5 ms.
static hb_status calibrate_one(hb_ctx* c, int kind, uint64_t probe_n, uint64_t steps, int repeats,
                               double* t, double* spread) {
    std::vector<uint64_t> seeds(probe_n);
    for (uint64_t i = 0; i < probe_n; ++i) seeds[i] = i;
    HB_TRY(validate(c, kind, seeds.data(), probe_n, steps, seeds.data()));
    if (c->fault_mode == HB_FAULT_DEVICE)
        return c->fail(HB_CUDA_ERROR, "injected device fault (hb_ctx_inject_fault)");
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    HB_TRY(stage_inputs(c, kind, seeds.data(), probe_n));
    cudaEvent_t e0, e1;
    HB_TRY(c->cuda(cudaEventCreate(&e0), "event"));
    if (cudaEventCreate(&e1) != cudaSuccess) {
        cudaEventDestroy(e0);
        return c->fail(HB_CUDA_ERROR, "event");
    }
    auto sample = [&](int k, double* ms) -> hb_status {
        HB_TRY(c->cuda(cudaEventRecord(e0, c->stream), "event record"));
        for (int j = 0; j < k; ++j)
            HB_TRY(launch(c, kind, probe_n, steps, hb::kSimDt, c->staged_from_seeds, nullptr));
        HB_TRY(c->cuda(cudaEventRecord(e1, c->stream), "event record"));
        HB_TRY(c->cuda(cudaEventSynchronize(e1), "event sync"));
        float f = 0.f;
        HB_TRY(c->cuda(cudaEventElapsedTime(&f, e0, e1), "event time"));
        *ms = static_cast<double>(f) / k;
        return HB_OK;
    };
    hb_status st = HB_OK;
    double one = 0.0;
    std::vector<double> v;
    if ((st = sample(1, &one)) == HB_OK && (st = sample(1, &one)) == HB_OK) {  // warm-up, then size
        const int k = static_cast<int>(std::min(4096.0, std::max(1.0, std::ceil(5.0 / std::max(one, 1e-4)))));
        for (int r = 0; r < repeats && st == HB_OK; ++r) {
            double ms = 0.0;
            st = sample(k, &ms);
            v.push_back(ms);
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->counters_dirty = true;  // the probe's launches added to the counters
    c->staged_kind = -1;
    if (st != HB_OK) return st;
    std::sort(v.begin(), v.end());
    const size_t m = v.size();
    const double med = m % 2 ? v[m / 2] : 0.5 * (v[m / 2 - 1] + v[m / 2]);
    *t = 1e-3 * med;
    *spread = med > 0.0 ? (v.back() - v.front()) / med : 0.0;
    return HB_OK;
}

hb_status hb_calibrate(hb_ctx* const* ctxs, int count, int kind, uint64_t probe_n, uint64_t steps,
                       int repeats, double* t_s, double* spread, int* ok) {
    if (!ctxs || count < 1 || !t_s || !ok || repeats < 1) return set_global(HB_INVALID_ARG, "bad arguments");
    if (probe_n < 1) return set_global(HB_INVALID_ARG, "calibrate: probe_n must be >= 1");
    if (!valid_kind(kind)) return set_global(HB_INVALID_ARG, "unknown model kind");
    if (steps < 1) return set_global(HB_INVALID_ARG, "batch request: steps must be >= 1");
    for (int d = 0; d < count; ++d)
        if (!ctxs[d]) return set_global(HB_INVALID_ARG, "null context");
    std::vector<double> sp(count, 0.0);
    std::vector<hb_status> st(count, HB_OK);
    for (int d = 0; d < count; ++d)
        worker_of(ctxs[d]).submit([&, d] {
            st[d] = calibrate_one(ctxs[d], kind, probe_n, steps, repeats, &t_s[d], &sp[d]);
        });
    int alive = 0;
    for (int d = 0; d < count; ++d) {
        worker_of(ctxs[d]).wait();
        ok[d] = st[d] == HB_OK;
        if (!ok[d]) t_s[d] = 0.0, sp[d] = 0.0;
        alive += ok[d];
        if (spread) spread[d] = sp[d];
    }
    if (!alive) return set_global(HB_CUDA_ERROR, "calibrate: all back-ends failed");
    return HB_OK;
}

int hb_snap_equal_times(const double* t_s, const double* spread, const int* ok, int count,
                        double min_rel_tol, double* out_t_s) {
    if (!t_s || !out_t_s || count < 1) return 0;
    double lo = 0.0, hi = 0.0, sum = 0.0, tol = min_rel_tol;
    int alive = 0;
    for (int d = 0; d < count; ++d) {
        out_t_s[d] = t_s[d];
        if (ok && !ok[d]) continue;
        if (!(t_s[d] > 0.0) || !std::isfinite(t_s[d])) return 0;
        lo = alive ? std::min(lo, t_s[d]) : t_s[d];
        hi = alive ? std::max(hi, t_s[d]) : t_s[d];
        sum += t_s[d];
        if (spread) tol = std::max(tol, spread[d]);
        ++alive;
    }
    if (alive < 2 || (hi - lo) / lo > tol) return 0;
    for (int d = 0; d < count; ++d)
        if (!ok || ok[d]) out_t_s[d] = sum / alive;
    return 1;
}

hb_status hb_fp64_peak(hb_ctx* c, double* ops_per_s, double* ms) {
    if (!c || !ops_per_s) return set_global(HB_INVALID_ARG, "bad arguments");
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double ops = 0.0;
    const int iters = 4096;
    hb::launch_fp64_probe(c->d_scratch, c->sms, iters, c->stream, &ops);  // warm-up
    cudaEventRecord(e0, c->stream);
    HB_TRY(c->cuda(hb::launch_fp64_probe(c->d_scratch, c->sms, iters, c->stream, &ops), "fp64 probe"));
    cudaEventRecord(e1, c->stream);
    HB_TRY(c->cuda(cudaEventSynchronize(e1), "event sync"));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ops_per_s = ops / (static_cast<double>(t) * 1e-3);
    if (ms) *ms = t;
    return HB_OK;
}


hb_status hb_check_fast_math(hb_ctx* c, const double* x, const double* y, size_t n,
                             uint64_t* sqrt_mismatch, uint64_t* div_mismatch,
                             uint64_t* sqrt_flagged, uint64_t* div_flagged) {
    if (!c || !x || !y || n == 0) return set_global(HB_INVALID_ARG, "bad arguments");
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    double* d = nullptr;
    unsigned char* fl = nullptr;
    HB_TRY(c->cuda(cudaMalloc(&d, 6 * n * sizeof(double)), "cudaMalloc"));
    if (cudaMalloc(&fl, n) != cudaSuccess) {
        cudaFree(d);
        return c->fail(HB_CUDA_ERROR, "cudaMalloc(flags)");
    }
    std::vector<double> o(4 * n);
    std::vector<unsigned char> f(n);
    cudaMemcpy(d, x, n * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(d + n, y, n * sizeof(double), cudaMemcpyHostToDevice);
    cudaError_t e = hb::launch_fastpath_check(d, d + n, n, d + 2 * n, d + 3 * n, d + 4 * n, d + 5 * n,
                                              fl, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = cudaMemcpy(o.data(), d + 2 * n, 4 * n * sizeof(double), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(f.data(), fl, n, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(fl);
    HB_TRY(c->cuda(e, "fast-math check"));
    uint64_t sm = 0, dm = 0, sf = 0, df = 0;
    for (size_t i = 0; i < n; ++i) {
        const bool fs = f[i] & 1, fd = f[i] & 2;
        sf += fs;
        df += fd;
        if (!fs && std::memcmp(&o[i], &o[n + i], 8) != 0) ++sm;
        if (!fd && std::memcmp(&o[2 * n + i], &o[3 * n + i], 8) != 0) ++dm;
    }
    if (sqrt_mismatch) *sqrt_mismatch = sm;
    if (div_mismatch) *div_mismatch = dm;
    if (sqrt_flagged) *sqrt_flagged = sf;
    if (div_flagged) *div_flagged = df;
    return HB_OK;
}

}  // extern "C"

// ===========================================================================
// Generation loop (host orchestration; kernels in hb_ea.cu)
namespace {

std::string batch_failure_text(const uint64_t* seeds, const uint64_t* fail, size_t n) {
    // executor.cpp:20-28 with failed() sorted by (seed, message)
    std::vector<std::pair<uint64_t, std::string>> failed;
    for (size_t i = 0; i < n; ++i)
        if (fail[i]) {
            char buf[256];
            hb_format_blowup(seeds[i], fail[i], hb::kSimDt, buf, sizeof buf);
            failed.emplace_back(seeds[i], buf);
        }
    if (failed.empty()) return "numerical blow-up in batch";
    std::sort(failed.begin(), failed.end());
    std::string msg = "batch failed for seed " + std::to_string(failed.front().first);
    if (failed.size() > 1) msg += " (+" + std::to_string(failed.size() - 1) + " more)";
    return msg + ": " + failed.front().second;
}

// The sequential std::max fold of ea.cpp:101-103 starting from `init` (the
// first of equal maxima, e.g. +0 before -0, wins; a NaN init stays) without
// its one dependent chain: eight independent running maxima, then the first
// element equal to the maximum.  Over a final population the parents are
// sorted descending, so the fold over all of it is the fold over the
// offspring starting from parent 0.
double fold_max(double init, const double* f, size_t n) {
    double m[8];
    for (double& v : m) v = init;
    size_t i = 0;
    for (; i + 8 <= n; i += 8)
        for (int k = 0; k < 8; ++k) m[k] = f[i + k] > m[k] ? f[i + k] : m[k];
    for (; i < n; ++i) m[0] = f[i] > m[0] ? f[i] : m[0];
    double mx = m[0];
    for (int k = 1; k < 8; ++k) mx = m[k] > mx ? m[k] : mx;
    if (init == mx) return init;
    for (size_t j = 0; j < n; ++j)
        if (f[j] == mx) return f[j];
    return init;
}

// The stepping launch of an evaluation (+ the fitness gather): the initial
// state is built from the seeds on the device (Box) or already in c->d_init.
hb_status eval_kernel(hb_ctx* c, int kind, const uint64_t* d_seeds, size_t n, uint64_t steps,
                      double* d_fitness) {
    const bool dev_init = init_on_device(c, kind);
    if (c->counters_dirty) {
        HB_TRY(c->cuda(cudaMemsetAsync(c->d_count, 0, 2 * sizeof(unsigned), c->stream), "memset(count)"));
        c->counters_dirty = false;
    }
    hb::SimArgs a{dev_init ? nullptr : c->d_init, d_seeds, n, n, steps, hb::kSimDt,
                  c->d_out, c->d_fail, c->d_count, nullptr, nullptr, c->d_ops};
    if (kind == hb::Box && c->kernel_variant == HB_KERNEL_AUTO) a.fitness = d_fitness;  // no records, no gather
    HB_TRY(c->cuda(launch_kernel(c, kind, a), "kernel launch"));
    if (!a.fitness)
        HB_TRY(c->cuda(hb::ea_fitness_from_results(c->d_out, n, d_fitness, c->stream), "fitness gather"));
    return HB_OK;
}

// Launch the simulation of n device-resident seeds on c's device; fitness
// lands in d_fitness (c's device).  Models initialised on the host take the
// seeds through the host initialiser first (blocking).  Counters are read
// back asynchronously; eval_finish synchronises and checks them.
hb_status eval_start(hb_ctx* c, int kind, const uint64_t* d_seeds, size_t n, uint64_t steps,
                     double* d_fitness, bool read_counts = true) {
    const bool dev_init = init_on_device(c, kind);
    HB_TRY(ensure_capacity(c, kind, n, !dev_init));
    if (!dev_init) {
        Trace tr("eval-init");
        HB_TRY(c->cuda(cudaMemcpyAsync(c->h_seeds, d_seeds, n * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                       c->stream), "D2H seeds"));
        HB_TRY(c->cuda(cudaStreamSynchronize(c->stream), "stream sync"));
        tr.mark("d2h_seeds+wait");
        double* soa = c->h_init;
        const uint64_t* hs = c->h_seeds;
        if (trig_init(c, kind)) {
            pool_of(c).run(n, [&](size_t b, size_t e) { trig_range(kind, hs, b, e, soa, n); }, 64);
            tr.mark("trig");
            const size_t rows = 2 * static_cast<size_t>(hb::init_angles(kind));
            HB_TRY(c->cuda(cudaMemcpyAsync(c->d_trig, c->h_init, rows * n * sizeof(double),
                                           cudaMemcpyHostToDevice, c->stream), "H2D trig"));
            HB_TRY(c->cuda(hb::launch_init(kind, d_seeds, c->d_trig, n, c->d_init, c->stream), "init kernel"));
        } else {
            pool_of(c).run(n, [&](size_t b, size_t e) { build_range(kind, hs, b, e, soa, n); }, 64);
            tr.mark("build");
            const size_t rows = static_cast<size_t>(hb::state_rows(kind));
            HB_TRY(c->cuda(cudaMemcpyAsync(c->d_init, c->h_init, rows * n * sizeof(double),
                                           cudaMemcpyHostToDevice, c->stream), "H2D init"));
        }
        tr.mark("h2d_enqueue");
    }
    HB_TRY(eval_kernel(c, kind, d_seeds, n, steps, d_fitness));
    if (read_counts)
        HB_TRY(c->cuda(cudaMemcpyAsync(c->h_count, c->d_count, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                                       c->stream), "D2H count"));
    return HB_OK;
}

hb_status eval_finish(hb_ctx* c, const uint64_t* d_seeds, size_t n, uint64_t* n_failed) {
    HB_TRY(c->cuda(cudaStreamSynchronize(c->stream), "stream sync"));
    c->last_failed = c->h_count[0];
    c->last_replays = c->h_count[1];
    c->counters_dirty = (c->h_count[0] | c->h_count[1]) != 0;
    if (n_failed) *n_failed = c->h_count[0];
    if (c->h_count[0] == 0) return HB_OK;
    std::vector<uint64_t> seeds(n), fail(n);
    HB_TRY(c->cuda(cudaMemcpy(seeds.data(), d_seeds, n * sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H"));
    HB_TRY(c->cuda(cudaMemcpy(fail.data(), c->d_fail, n * sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H"));
    return c->fail(HB_BLOWUP_PARTIAL, batch_failure_text(seeds.data(), fail.data(), n));
}

void enable_peer(int a, int b) {
    if (a == b) return;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, a, b);
    if (can) {
        cudaSetDevice(a);
        if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
    }
}

// Evaluate seeds src[0, n) living on ctxs[0]'s device, sharded over the
// contexts; fitness into dst[0, n) on ctxs[0]'s device.  `ready` is an event
// on ctxs[0]'s stream after which src is valid.
hb_status eval_sharded(hb_ctx* const* ctxs, int count, const std::vector<uint64_t>& shares, int kind,
                       const uint64_t* src, size_t n, uint64_t steps, double* dst, cudaEvent_t ready) {
    if (count == 1) {  // one device: no helper thread
        hb_ctx* c = ctxs[0];
        HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
        HB_TRY(eval_start(c, kind, src, n, steps, dst));
        return eval_finish(c, src, n, nullptr);
    }
    std::vector<hb_status> st(count, HB_OK);
    std::vector<std::string> err(count);
    std::vector<int> busy;
    size_t begin = 0;
    for (int d = 0; d < count; ++d) {
        const size_t b = begin, len = shares[d];
        begin += len;
        if (len == 0) continue;
        busy.push_back(d);
        worker_of(ctxs[d]).submit([&, d, b, len] {
            hb_ctx* c = ctxs[d];
            auto run = [&]() -> hb_status {
                HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
                if (d == 0) {
                    HB_TRY(eval_start(c, kind, src + b, len, steps, dst + b));
                    return eval_finish(c, src + b, len, nullptr);
                }
                HB_TRY(ensure_capacity(c, kind, len, false));
                HB_TRY(grow_dev(c, &c->d_ea_fit, c->d_ea_fit_cap, len, "cudaMalloc(ea fit)"));
                HB_TRY(c->cuda(cudaStreamWaitEvent(c->stream, ready, 0), "wait"));
                HB_TRY(c->cuda(cudaMemcpyPeerAsync(c->d_seeds, c->device, src + b, ctxs[0]->device,
                                                   len * sizeof(uint64_t), c->stream), "peer seeds"));
                HB_TRY(eval_start(c, kind, c->d_seeds, len, steps, c->d_ea_fit));
                HB_TRY(c->cuda(cudaMemcpyPeerAsync(dst + b, ctxs[0]->device, c->d_ea_fit, c->device,
                                                   len * sizeof(double), c->stream), "peer fitness"));
                return eval_finish(c, c->d_seeds, len, nullptr);
            };
            st[d] = run();
            if (st[d] != HB_OK) err[d] = c->err;
        });
    }
    for (int d : busy) worker_of(ctxs[d]).wait();
    for (int d = 0; d < count; ++d)
        if (st[d] != HB_OK) return ctxs[0]->fail(st[d], err[d]);
    return HB_OK;
}

// Spin (briefly), then yield, until `a` reaches `v`: host-side ordering of
// the enqueues of the queued multi-context loop (a stream may only wait on an
// event after the event's record has been enqueued).
void wait_at_least(const std::atomic<uint64_t>& a, uint64_t v) {
    for (int i = 0; a.load(std::memory_order_acquire) < v; ++i)
        if (i > 2000) std::this_thread::yield();
}

hb_status ensure_events(hb_ctx* c, std::vector<cudaEvent_t>& ev, size_t n, unsigned flags) {
    while (ev.size() < n) {
        cudaEvent_t e;
        HB_TRY(c->cuda(cudaEventCreateWithFlags(&e, flags), "event"));
        ev.push_back(e);
    }
    return HB_OK;
}

// The generation loop over `count` contexts, queued: no host synchronisation
// per generation for device-initialised models (Box) and exactly one (the
// offspring seeds for the host's libm cos / sin) for the others.  Device 0
// holds the population and runs the selection graph; every device d
// evaluates its contiguous slice of each evaluation (shares from the
// splitter) on its own stream, driven by its persistent worker thread:
//   dev d: wait(sel[g]) -> seeds slice in (peer copy) -> [init] -> kernel ->
//          fitness slice out (peer copy into device 0's population) -> done[d][g]
//   dev 0: wait(done[*][g-1]) -> selection graph -> sel[g] -> own slice
// The host threads only order their enqueues (an event must be recorded
// before a stream waits on it); all data dependencies are stream / event
// ordered on the devices.  Failure counters accumulate over the loop and are
// read once at the end: *any_fail tells the caller to re-run checked.
hb_status run_ea_queued(hb_ctx* const* ctxs, int count, int kind, size_t pop, uint64_t G, uint64_t steps,
                        uint64_t seed, const std::vector<uint64_t>& sh_pop, const std::vector<uint64_t>& sh_mu,
                        uint64_t* const d_gen[2], double* const d_fit[2], uint64_t* genomes_out,
                        double* fitness_out, double* best_out, hb_phase_profile* prof_out, bool* any_fail) {
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    hb_ctx* c0 = ctxs[0];
    const size_t mu = pop / 2;
    const bool dev_init = init_on_device(c0, kind);
    const int J2 = 2 * hb::init_angles(kind);  // trig rows (host-initialised kinds)
    // slices: evaluation g covers [off_g, off_g + n_g) of buffer g & 1
    std::vector<std::vector<size_t>> beg(2, std::vector<size_t>(count + 1, 0));
    for (int d = 0; d < count; ++d) {
        beg[0][d + 1] = beg[0][d] + sh_pop[d];
        beg[1][d + 1] = beg[1][d] + sh_mu[d];
    }
    auto n_of = [&](uint64_t g) { return g == 0 ? pop : mu; };
    auto off_of = [&](uint64_t g) { return g == 0 ? size_t{0} : mu; };
    auto b_of = [&](uint64_t g, int d) { return beg[g == 0 ? 0 : 1][d]; };
    auto len_of = [&](uint64_t g, int d) { return g == 0 ? sh_pop[d] : sh_mu[d]; };

    // capacities and events (synchronous allocations happen here, up front)
    for (int d = 0; d < count; ++d) {
        hb_ctx* c = ctxs[d];
        const size_t cap = std::max<size_t>(std::max(sh_pop[d], sh_mu[d]), d == 0 && !dev_init ? pop : 1);
        HB_TRY(ensure_capacity(c, kind, cap, !dev_init));
        HB_TRY(grow_dev(c, &c->d_ea_fit, c->d_ea_fit_cap, cap, "cudaMalloc(ea fit)"));
        HB_TRY(ensure_events(c, c->ea_chain, G + 1, cudaEventDisableTiming));
        if (c->counters_dirty) {
            HB_TRY(c->cuda(cudaMemsetAsync(c->d_count, 0, 2 * sizeof(unsigned), c->stream), "memset(count)"));
            c->counters_dirty = false;
        }
    }
    HB_TRY(c0->cuda(cudaSetDevice(c0->device), "cudaSetDevice"));
    HB_TRY(ensure_events(c0, c0->ea_timing, 2 * G + 2, cudaEventDefault));
    if (!c0->ea_copy) {
        HB_TRY(c0->cuda(cudaStreamCreateWithFlags(&c0->ea_copy, cudaStreamNonBlocking), "stream"));
        HB_TRY(c0->cuda(cudaEventCreateWithFlags(&c0->ea_sel_done, cudaEventDisableTiming), "event"));
    }
    cudaEvent_t* tev = c0->ea_timing.data();
    cudaEvent_t* sel = c0->ea_chain.data();  // sel[g]: population g is ready on device 0

    std::atomic<uint64_t> posted{0};  // sel[g] (Box) / host trig rows of g (others) recorded for g < posted
    std::vector<std::atomic<uint64_t>> done(count);
    for (auto& x : done) x.store(0);
    std::atomic<int> abort{0};
    std::vector<hb_status> st(count, HB_OK);
    std::vector<std::string> err(count);

    // one evaluation slice on context c (d >= 1: through c's own buffers)
    auto slice = [&](int d, uint64_t g) -> hb_status {
        hb_ctx* c = ctxs[d];
        const size_t n = n_of(g), b = b_of(g, d), len = len_of(g, d);
        uint64_t* src = d_gen[g & 1] + off_of(g) + b;
        double* dst = d_fit[g & 1] + off_of(g) + b;
        if (len == 0) return HB_OK;
        const uint64_t* seeds = src;
        if (!dev_init) {  // seeds and cos / sin rows from device 0's pinned staging
            HB_TRY(c->cuda(cudaMemcpyAsync(c->d_seeds, c0->h_seeds + b, len * sizeof(uint64_t),
                                           cudaMemcpyHostToDevice, c->stream), "H2D seeds"));
            HB_TRY(c->cuda(cudaMemcpy2DAsync(c->d_trig, len * sizeof(double), c0->h_init + b, n * sizeof(double),
                                             len * sizeof(double), J2, cudaMemcpyHostToDevice, c->stream),
                           "H2D trig"));
            HB_TRY(c->cuda(hb::launch_init(kind, c->d_seeds, c->d_trig, len, c->d_init, c->stream), "init kernel"));
            seeds = c->d_seeds;
        } else if (d > 0) {
            HB_TRY(c->cuda(cudaMemcpyPeerAsync(c->d_seeds, c->device, src, c0->device, len * sizeof(uint64_t),
                                               c->stream), "peer seeds"));
            seeds = c->d_seeds;
        }
        if (d == 0) return eval_kernel(c, kind, seeds, len, steps, dst);
        HB_TRY(eval_kernel(c, kind, seeds, len, steps, c->d_ea_fit));
        return c->cuda(cudaMemcpyPeerAsync(dst, c0->device, c->d_ea_fit, c->device, len * sizeof(double),
                                           c->stream), "peer fitness");
    };
    for (int d = 1; d < count; ++d) {
        if (sh_pop[d] == 0 && sh_mu[d] == 0) {
            done[d].store(G + 1);
            continue;
        }
        worker_of(ctxs[d]).submit([&, d] {
            hb_ctx* c = ctxs[d];
            auto run = [&]() -> hb_status {
                HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
                for (uint64_t g = 0; g <= G; ++g) {
                    wait_at_least(posted, g + 1);
                    if (abort.load()) return HB_OK;
                    if (dev_init) HB_TRY(c->cuda(cudaStreamWaitEvent(c->stream, sel[g], 0), "wait"));
                    HB_TRY(slice(d, g));
                    HB_TRY(c->cuda(cudaEventRecord(c->ea_chain[g], c->stream), "record"));
                    done[d].store(g + 1, std::memory_order_release);
                }
                return HB_OK;
            };
            st[d] = run();
            if (st[d] != HB_OK) {
                err[d] = c->err;
                abort.store(1);
                done[d].store(G + 1);
            }
        });
    }
    // device 0 (this thread)
    auto host_rows = [&](uint64_t g) -> hb_status {  // offspring seeds to the host, libm cos / sin rows
        const size_t n = n_of(g);
        HB_TRY(c0->cuda(cudaMemcpyAsync(c0->h_seeds, d_gen[g & 1] + off_of(g), n * sizeof(uint64_t),
                                        cudaMemcpyDeviceToHost, c0->stream), "D2H seeds"));
        HB_TRY(c0->cuda(cudaStreamSynchronize(c0->stream), "stream sync"));
        const uint64_t* hs = c0->h_seeds;
        double* trig = c0->h_init;
        pool_of(c0).run(n, [&](size_t b, size_t e) { trig_range(kind, hs, b, e, trig, n); }, 64);
        return HB_OK;
    };
    auto main_loop = [&]() -> hb_status {
        HB_TRY(c0->cuda(cudaEventRecord(tev[0], c0->stream), "record"));
        HB_TRY(c0->cuda(hb::ea_init_genomes(seed, pop, d_gen[0], c0->stream, c0->d_ea_g), "init genomes"));
        for (uint64_t g = 0; g <= G; ++g) {
            if (g > 0) {
                for (int d = 1; d < count; ++d) {
                    if (len_of(g - 1, d) == 0) continue;
                    wait_at_least(done[d], g);
                    if (abort.load()) return HB_OK;
                    HB_TRY(c0->cuda(cudaStreamWaitEvent(c0->stream, ctxs[d]->ea_chain[g - 1], 0), "wait"));
                }
                HB_TRY(c0->cuda(cudaEventRecord(tev[2 * g], c0->stream), "record"));
                HB_TRY(c0->cuda(cudaGraphLaunch(c0->ea_graph[(g - 1) & 1], c0->stream), "select/vary"));
                HB_TRY(c0->cuda(cudaEventRecord(tev[2 * g + 1], c0->stream), "record"));
                if (g == G) {  // final genomes + parent fitness out while the offspring evaluate
                    const bool pg = is_pinned(genomes_out), pf = is_pinned(fitness_out);
                    HB_TRY(c0->cuda(cudaEventRecord(c0->ea_sel_done, c0->stream), "record"));
                    HB_TRY(c0->cuda(cudaStreamWaitEvent(c0->ea_copy, c0->ea_sel_done, 0), "wait"));
                    HB_TRY(c0->cuda(cudaMemcpyAsync(pg ? genomes_out : c0->h_ea_gen, d_gen[G & 1],
                                                    pop * sizeof(uint64_t), cudaMemcpyDeviceToHost, c0->ea_copy),
                                    "D2H"));
                    HB_TRY(c0->cuda(cudaMemcpyAsync(pf ? fitness_out : c0->h_ea_fit, d_fit[G & 1],
                                                    mu * sizeof(double), cudaMemcpyDeviceToHost, c0->ea_copy),
                                    "D2H"));
                }
            }
            if (!dev_init) HB_TRY(host_rows(g));
            HB_TRY(c0->cuda(cudaEventRecord(sel[g], c0->stream), "record"));
            posted.store(g + 1, std::memory_order_release);
            HB_TRY(slice(0, g));
        }
        for (int d = 1; d < count; ++d) {
            if (len_of(G, d) == 0) continue;
            wait_at_least(done[d], G + 1);
            if (abort.load()) return HB_OK;
            HB_TRY(c0->cuda(cudaStreamWaitEvent(c0->stream, ctxs[d]->ea_chain[G], 0), "wait"));
        }
        return c0->cuda(cudaEventRecord(tev[1], c0->stream), "record");
    };
    hb_status st0 = main_loop();
    if (st0 != HB_OK) {
        abort.store(1);
        posted.store(G + 2);
    }
    for (int d = 1; d < count; ++d)
        if (sh_pop[d] || sh_mu[d]) worker_of(ctxs[d]).wait();
    const auto t_enq = clk::now();
    if (st0 != HB_OK) return st0;
    for (int d = 1; d < count; ++d)
        if (st[d] != HB_OK) return c0->fail(st[d], "device " + std::to_string(d) + ": " + err[d]);
    // results: offspring fitness of the last generation, then every device's
    // accumulated failure counter
    const bool pg = is_pinned(genomes_out), pf = is_pinned(fitness_out);
    double* h_fit = pf ? fitness_out : c0->h_ea_fit;
    HB_TRY(c0->cuda(cudaMemcpyAsync(h_fit + mu, d_fit[G & 1] + mu, mu * sizeof(double), cudaMemcpyDeviceToHost,
                                    c0->stream), "D2H"));
    uint64_t failed = 0;
    for (int d = 0; d < count; ++d) {
        hb_ctx* c = ctxs[d];
        HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
        HB_TRY(c->cuda(cudaMemcpyAsync(c->h_count, c->d_count, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                                       c->stream), "D2H count"));
    }
    for (int d = 0; d < count; ++d) {
        hb_ctx* c = ctxs[d];
        HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
        HB_TRY(c->cuda(cudaStreamSynchronize(c->stream), "sync"));
        c->last_failed = c->h_count[0];
        c->last_replays = c->h_count[1];
        c->counters_dirty = (c->h_count[0] | c->h_count[1]) != 0;
        failed += c->h_count[0];
    }
    HB_TRY(c0->cuda(cudaSetDevice(c0->device), "cudaSetDevice"));
    HB_TRY(c0->cuda(cudaStreamSynchronize(c0->ea_copy), "sync"));
    *any_fail = failed != 0;
    if (*any_fail) return HB_OK;
    if (!pg) std::memcpy(genomes_out, c0->h_ea_gen, pop * sizeof(uint64_t));
    if (!pf) std::memcpy(fitness_out, c0->h_ea_fit, pop * sizeof(double));
    if (best_out) *best_out = fold_max(fitness_out[0], fitness_out + mu, mu);
    hb_phase_profile prof{};
    float ms = 0.f;
    double sel_s = 0.0;
    for (uint64_t g = 1; g <= G; ++g) {
        cudaEventElapsedTime(&ms, tev[2 * g], tev[2 * g + 1]);
        sel_s += 1e-3 * ms;
    }
    cudaEventElapsedTime(&ms, tev[0], tev[1]);
    const double span = 1e-3 * ms;
    prof.total_s = elapsed_s(t_start);
    prof.selection_s = std::min(sel_s, prof.total_s);
    prof.evaluation_s = std::min(std::max(span - sel_s, 0.0), prof.total_s - prof.selection_s);
    prof.bookkeeping_s = prof.total_s - prof.selection_s - prof.evaluation_s;
    prof.host_overhead_s = std::max(0.0, prof.total_s - span);
    (void)t_enq;
    *prof_out = prof;
    return HB_OK;
}

}  // namespace

extern "C" {

hb_status hb_eval_device(hb_ctx* c, int kind, const uint64_t* d_seeds, size_t n, uint64_t steps,
                         double* d_fitness, uint64_t* n_failed) {
    if (!c) return set_global(HB_INVALID_ARG, "null context");
    HB_TRY(validate(c, kind, d_seeds, n, steps, d_fitness));
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    HB_TRY(eval_start(c, kind, d_seeds, n, steps, d_fitness));
    return eval_finish(c, d_seeds, n, n_failed);
}

hb_status hb_ea_init_genomes(hb_ctx* c, uint64_t seed, size_t pop, uint64_t* d_genomes) {
    if (!c || !d_genomes) return set_global(HB_INVALID_ARG, "bad arguments");
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    return c->cuda(hb::ea_init_genomes(seed, pop, d_genomes, c->stream), "init genomes");
}

hb_status hb_ea_select_vary(hb_ctx* c, const uint64_t* d_genomes, const double* d_fitness, size_t pop,
                            uint64_t g, uint64_t* d_next, double* d_next_fitness) {
    if (!c || !d_genomes || !d_fitness || !d_next || !d_next_fitness)
        return set_global(HB_INVALID_ARG, "bad arguments");
    if (pop < 2 || pop % 2) return c->fail(HB_INVALID_ARG, "run_ea: population_size must be even and >= 2");
    HB_TRY(c->cuda(cudaSetDevice(c->device), "cudaSetDevice"));
    const size_t bytes = hb::ea_select_scratch_bytes(pop);
    if (bytes > c->d_ea_scratch_cap) {  // the context's persistent selection scratch
        HB_TRY(c->cuda(cudaStreamSynchronize(c->stream), "stream sync"));
        cudaFree(c->d_ea_scratch);
        c->d_ea_scratch = nullptr;
        c->d_ea_scratch_cap = 0;
        for (cudaGraphExec_t& ge : c->ea_graph) {  // captured against the old scratch
            if (ge) cudaGraphExecDestroy(ge);
            ge = nullptr;
        }
        c->ea_graph_pop = 0;
        HB_TRY(c->cuda(cudaMalloc(&c->d_ea_scratch, bytes), "cudaMalloc(ea scratch)"));
        c->d_ea_scratch_cap = bytes;
    }
    return c->cuda(hb::ea_select_vary(d_genomes, d_fitness, pop, g, d_next, d_next_fitness, c->d_ea_scratch,
                                      c->d_ea_scratch_cap, c->stream),
                   "select/vary");
}

hb_status hb_run_ea(hb_ctx* const* ctxs, int count, const double* device_times, int kind, size_t pop,
                    uint64_t generations, uint64_t steps, uint64_t seed, uint64_t* genomes_out,
                    double* fitness_out, double* best_out, hb_phase_profile* profile,
                    uint64_t* history_genomes, double* history_fitness) {
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    if (!ctxs || count < 1 || !ctxs[0]) return set_global(HB_INVALID_ARG, "no contexts");
    hb_ctx* c0 = ctxs[0];
    if (!valid_kind(kind)) return c0->fail(HB_INVALID_ARG, "unknown model kind");
    if (pop < 2 || pop % 2 != 0) return c0->fail(HB_INVALID_ARG, "run_ea: population_size must be even and >= 2");
    if (generations < 1) return c0->fail(HB_INVALID_ARG, "run_ea: generations must be >= 1");
    if (steps < 1) return c0->fail(HB_INVALID_ARG, "batch request: steps must be >= 1");
    if (!genomes_out || !fitness_out) return c0->fail(HB_INVALID_ARG, "null output");
    hb_phase_profile prof{};
    for (int d = 1; d < count; ++d) {
        enable_peer(ctxs[0]->device, ctxs[d]->device);
        enable_peer(ctxs[d]->device, ctxs[0]->device);
    }
    HB_TRY(c0->cuda(cudaSetDevice(c0->device), "cudaSetDevice"));
    const size_t mu = pop / 2;
    const size_t scratch_bytes = hb::ea_select_scratch_bytes(pop);
    if (pop > c0->d_ea_pop_cap) {
        for (int k = 0; k < 2; ++k) {
            cudaFree(c0->d_ea_gen[k]); cudaFree(c0->d_ea_pfit[k]);
            c0->d_ea_gen[k] = nullptr; c0->d_ea_pfit[k] = nullptr;
        }
        cudaFreeHost(c0->h_ea_gen); cudaFreeHost(c0->h_ea_fit);
        c0->h_ea_gen = nullptr; c0->h_ea_fit = nullptr;
        c0->d_ea_pop_cap = 0;
        for (int k = 0; k < 2; ++k) {
            HB_TRY(c0->cuda(cudaMalloc(&c0->d_ea_gen[k], pop * sizeof(uint64_t)), "cudaMalloc(ea genomes)"));
            HB_TRY(c0->cuda(cudaMalloc(&c0->d_ea_pfit[k], pop * sizeof(double)), "cudaMalloc(ea fitness)"));
        }
        HB_TRY(c0->cuda(cudaHostAlloc(&c0->h_ea_gen, pop * sizeof(uint64_t), 0), "cudaHostAlloc(ea)"));
        HB_TRY(c0->cuda(cudaHostAlloc(&c0->h_ea_fit, pop * sizeof(double), 0), "cudaHostAlloc(ea)"));
        c0->d_ea_pop_cap = pop;
    }
    if (c0->ea_graph_pop != pop || scratch_bytes > c0->d_ea_scratch_cap) {
        for (cudaGraphExec_t& g : c0->ea_graph) {
            if (g) cudaGraphExecDestroy(g);
            g = nullptr;
        }
        c0->ea_graph_pop = 0;
    }
    if (scratch_bytes > c0->d_ea_scratch_cap) {
        cudaFree(c0->d_ea_scratch);
        c0->d_ea_scratch = nullptr;
        c0->d_ea_scratch_cap = 0;
        HB_TRY(c0->cuda(cudaMalloc(&c0->d_ea_scratch, scratch_bytes), "cudaMalloc(ea scratch)"));
        c0->d_ea_scratch_cap = scratch_bytes;
    }
    if (!c0->ea_ev[0]) {
        HB_TRY(c0->cuda(cudaEventCreateWithFlags(&c0->ea_ev[0], cudaEventDisableTiming), "event"));
        HB_TRY(c0->cuda(cudaEventCreate(&c0->ea_ev[1]), "event"));
        HB_TRY(c0->cuda(cudaEventCreate(&c0->ea_ev[2]), "event"));
    }
    uint64_t* d_gen[2] = {c0->d_ea_gen[0], c0->d_ea_gen[1]};
    double* d_fit[2] = {c0->d_ea_pfit[0], c0->d_ea_pfit[1]};
    void* scratch = c0->d_ea_scratch;
    if (!c0->d_ea_g) HB_TRY(c0->cuda(cudaMalloc(&c0->d_ea_g, sizeof(uint64_t)), "cudaMalloc(ea g)"));
    if (c0->ea_graph_pop != pop) {
        for (int k = 0; k < 2; ++k)
            HB_TRY(c0->cuda(hb::ea_select_vary_graph(d_gen[k], d_fit[k], pop, c0->d_ea_g, d_gen[k ^ 1],
                                                     d_fit[k ^ 1], scratch, c0->d_ea_scratch_cap,
                                                     c0->stream, &c0->ea_graph[k]),
                            "capture select/vary"));
        c0->ea_graph_pop = pop;
    }
    cudaEvent_t ev_ready = c0->ea_ev[0], e0 = c0->ea_ev[1], e2 = c0->ea_ev[2];

    // a non-finite or non-positive device time marks a device without a
    // share (dead to the splitter, as a failed calibration)
    std::vector<double> times(count, 1.0);
    std::vector<int> alive(count, 1);
    if (device_times)
        for (int d = 0; d < count; ++d) {
            times[d] = device_times[d];
            alive[d] = std::isfinite(times[d]) && times[d] > 0.0;
        }
    if (std::find(alive.begin(), alive.end(), 1) == alive.end())
        return c0->fail(HB_INVALID_ARG, "run_ea: no device has a finite positive time");
    auto shares_for = [&](size_t n) {
        std::vector<uint64_t> sh(count);
        hb_plan_allocation_n(times.data(), alive.data(), count, n, sh.data());
        return sh;
    };
    auto snapshot = [&](int cur, uint64_t g) -> hb_status {
        if (!history_genomes && !history_fitness) return HB_OK;
        if (history_genomes)
            HB_TRY(c0->cuda(cudaMemcpyAsync(history_genomes + g * pop, d_gen[cur], pop * sizeof(uint64_t),
                                            cudaMemcpyDeviceToHost, c0->stream), "D2H history"));
        if (history_fitness)
            HB_TRY(c0->cuda(cudaMemcpyAsync(history_fitness + g * pop, d_fit[cur], pop * sizeof(double),
                                            cudaMemcpyDeviceToHost, c0->stream), "D2H history"));
        return c0->cuda(cudaStreamSynchronize(c0->stream), "sync");
    };

    // One device, seeds initialised on the device, no history requested: the
    // whole loop is queued on the stream with no host round trip per
    // generation.  The failure counter is not reset between evaluations, so
    // one read at the end covers all of them; a blow-up anywhere falls through
    // to the checked loop below, which re-runs from generation 0
    // (deterministic) and throws at the first failing batch exactly like
    // ea.cpp:81-82.
    if (count == 1 && !history_genomes && !history_fitness && init_on_device(c0, kind)) {
        const size_t n_ev = 2 * generations + 2;
        while (c0->ea_timing.size() < n_ev) {
            cudaEvent_t ev;
            HB_TRY(c0->cuda(cudaEventCreate(&ev), "event"));
            c0->ea_timing.push_back(ev);
        }
        if (!c0->ea_copy) {
            HB_TRY(c0->cuda(cudaStreamCreateWithFlags(&c0->ea_copy, cudaStreamNonBlocking), "stream"));
            HB_TRY(c0->cuda(cudaEventCreateWithFlags(&c0->ea_sel_done, cudaEventDisableTiming), "event"));
        }
        const bool pg = is_pinned(genomes_out), pf = is_pinned(fitness_out);
        uint64_t* h_gen = pg ? genomes_out : c0->h_ea_gen;
        double* h_fit = pf ? fitness_out : c0->h_ea_fit;
        cudaEvent_t* tev = c0->ea_timing.data();
        cudaEventRecord(tev[0], c0->stream);
        HB_TRY(c0->cuda(hb::ea_init_genomes(seed, pop, d_gen[0], c0->stream, c0->d_ea_g), "init genomes"));
        HB_TRY(eval_start(c0, kind, d_gen[0], pop, steps, d_fit[0], false));
        int q = 0;
        for (uint64_t g = 1; g <= generations; ++g) {
            const int nxt = q ^ 1;
            cudaEventRecord(tev[2 * g], c0->stream);
            HB_TRY(c0->cuda(cudaGraphLaunch(c0->ea_graph[q], c0->stream), "select/vary"));
            cudaEventRecord(tev[2 * g + 1], c0->stream);
            if (g == generations) {  // the final genomes and parent fitness are known: copy them
                cudaEventRecord(c0->ea_sel_done, c0->stream);  // out while the offspring evaluate
                HB_TRY(c0->cuda(cudaStreamWaitEvent(c0->ea_copy, c0->ea_sel_done, 0), "wait"));
                HB_TRY(c0->cuda(cudaMemcpyAsync(h_gen, d_gen[nxt], pop * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                                c0->ea_copy), "D2H"));
                HB_TRY(c0->cuda(cudaMemcpyAsync(h_fit, d_fit[nxt], mu * sizeof(double), cudaMemcpyDeviceToHost,
                                                c0->ea_copy), "D2H"));
            }
            HB_TRY(eval_start(c0, kind, d_gen[nxt] + mu, mu, steps, d_fit[nxt] + mu, false));
            q = nxt;
        }
        cudaEventRecord(tev[1], c0->stream);
        HB_TRY(c0->cuda(cudaMemcpyAsync(c0->h_count, c0->d_count, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                                        c0->stream), "D2H count"));
        HB_TRY(c0->cuda(cudaMemcpyAsync(h_fit + mu, d_fit[q] + mu, mu * sizeof(double), cudaMemcpyDeviceToHost,
                                        c0->stream), "D2H"));
        HB_TRY(c0->cuda(cudaStreamSynchronize(c0->stream), "sync"));
        HB_TRY(c0->cuda(cudaStreamSynchronize(c0->ea_copy), "sync"));
        c0->last_failed = c0->h_count[0];
        c0->last_replays = c0->h_count[1];
        c0->counters_dirty = (c0->h_count[0] | c0->h_count[1]) != 0;
        if (c0->h_count[0] == 0) {
            if (!pg) std::memcpy(genomes_out, c0->h_ea_gen, pop * sizeof(uint64_t));
            if (!pf) std::memcpy(fitness_out, c0->h_ea_fit, pop * sizeof(double));
            if (best_out) {
                *best_out = fold_max(fitness_out[0], fitness_out + mu, mu);
            }
            float ms = 0.f;
            double sel = 0.0;
            for (uint64_t g = 1; g <= generations; ++g) {
                cudaEventElapsedTime(&ms, tev[2 * g], tev[2 * g + 1]);
                sel += 1e-3 * ms;
            }
            cudaEventElapsedTime(&ms, tev[0], tev[1]);
            prof.total_s = elapsed_s(t_start);
            prof.selection_s = std::min(sel, prof.total_s);
            prof.evaluation_s = std::min(std::max(1e-3 * ms - sel, 0.0), prof.total_s - prof.selection_s);
            prof.bookkeeping_s = prof.total_s - prof.selection_s - prof.evaluation_s;
            prof.host_overhead_s = std::max(0.0, prof.total_s - 1e-3 * ms);
            if (profile) *profile = prof;
            return HB_OK;
        }
    }

    // Several contexts (or a host-initialised model): the queued
    // multi-context loop — persistent per-device workers, event-chained
    // generations, one host round trip per generation only for the libm
    // cos / sin of multi-body offspring.  A blow-up anywhere falls through to
    // the checked loop below, which reports it exactly.
    bool uniform = true;
    for (int d = 0; d < count; ++d)
        uniform = uniform && ctxs[d] && ctxs[d]->kernel_variant == c0->kernel_variant &&
                  ctxs[d]->precision == c0->precision;
    if (uniform && !history_genomes && !history_fitness && !(count == 1 && init_on_device(c0, kind)) &&
        (init_on_device(c0, kind) || trig_init(c0, kind))) {
        bool any = false;
        hb_phase_profile qp{};
        HB_TRY(run_ea_queued(ctxs, count, kind, pop, generations, steps, seed, shares_for(pop), shares_for(mu),
                             d_gen, d_fit, genomes_out, fitness_out, best_out, &qp, &any));
        if (!any) {
            qp.total_s = elapsed_s(t_start);
            qp.bookkeeping_s = std::max(0.0, qp.total_s - qp.selection_s - qp.evaluation_s);
            if (profile) *profile = qp;
            return HB_OK;
        }
        HB_TRY(c0->cuda(cudaSetDevice(c0->device), "cudaSetDevice"));
    }

    // initial population + evaluation (ea.cpp:48-54)
    auto tb = clk::now();
    HB_TRY(c0->cuda(hb::ea_init_genomes(seed, pop, d_gen[0], c0->stream, c0->d_ea_g), "init genomes"));
    cudaEventRecord(ev_ready, c0->stream);
    prof.bookkeeping_s += elapsed_s(tb);
    auto te = clk::now();
    HB_TRY(eval_sharded(ctxs, count, shares_for(pop), kind, d_gen[0], pop, steps, d_fit[0], ev_ready));
    prof.evaluation_s += elapsed_s(te);
    HB_TRY(snapshot(0, 0));

    int cur = 0;
    for (uint64_t g = 1; g <= generations; ++g) {
        const int nxt = cur ^ 1;
        // selection + variation on device 0 (ea.cpp:60-79)
        auto ts = clk::now();
        HB_TRY(c0->cuda(cudaSetDevice(c0->device), "cudaSetDevice"));
        cudaEventRecord(e0, c0->stream);
        const cudaError_t e = cudaGraphLaunch(c0->ea_graph[cur], c0->stream);  // generation g (device counter)
        cudaEventRecord(e2, c0->stream);
        cudaEventRecord(ev_ready, c0->stream);
        HB_TRY(c0->cuda(e, "select/vary"));
        // evaluate the offspring (ea.cpp:81-82); stream-ordered after the
        // selection (device 0's stream, or a wait on ev_ready elsewhere) —
        // the one host synchronisation per generation is the evaluation's
        HB_TRY(eval_sharded(ctxs, count, shares_for(mu), kind, d_gen[nxt] + mu, mu, steps, d_fit[nxt] + mu,
                            ev_ready));
        // split the host interval by the selection's device time (e0 -> e2)
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e2);
        const double span = elapsed_s(ts), sel = std::min(span, 1e-3 * ms);
        prof.selection_s += sel;
        prof.evaluation_s += span - sel;
        cur = nxt;
        HB_TRY(snapshot(cur, g));
    }
    // final population to the host
    tb = clk::now();
    HB_TRY(c0->cuda(cudaSetDevice(c0->device), "cudaSetDevice"));
    {
        const bool pg = is_pinned(genomes_out), pf = is_pinned(fitness_out);
        HB_TRY(c0->cuda(cudaMemcpyAsync(pg ? genomes_out : c0->h_ea_gen, d_gen[cur], pop * sizeof(uint64_t),
                                        cudaMemcpyDeviceToHost, c0->stream), "D2H"));
        HB_TRY(c0->cuda(cudaMemcpyAsync(pf ? fitness_out : c0->h_ea_fit, d_fit[cur], pop * sizeof(double),
                                        cudaMemcpyDeviceToHost, c0->stream), "D2H"));
        HB_TRY(c0->cuda(cudaStreamSynchronize(c0->stream), "sync"));
        if (!pg) std::memcpy(genomes_out, c0->h_ea_gen, pop * sizeof(uint64_t));
        if (!pf) std::memcpy(fitness_out, c0->h_ea_fit, pop * sizeof(double));
    }
    prof.bookkeeping_s += elapsed_s(tb);
    if (best_out) {
        *best_out = fold_max(fitness_out[0], fitness_out + mu, mu);
    }
    prof.total_s = elapsed_s(t_start);
    // the device time of selection+variation is reported as selection (one
    // graph: sort + gather + offspring); host time beyond the named phases
    // is bookkeeping (ea.cpp:95-97)
    const double accounted = prof.selection_s + prof.variation_s + prof.evaluation_s + prof.bookkeeping_s;
    if (prof.total_s > accounted) prof.bookkeeping_s += prof.total_s - accounted;
    if (profile) *profile = prof;
    return HB_OK;
}

}  // extern "C"
