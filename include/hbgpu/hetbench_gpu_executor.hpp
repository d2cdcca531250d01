// hetbench_gpu_executor.hpp — the reference-side binding of the B200 backend.
//
// Header-only adapter a hetbench maintainer adds to the reference build
// (see INTEGRATION.md).  It derives from the reference's own
// hetbench::batch_executor (proj/include/hetbench/executor.hpp:68-73) and
// forwards run() to the C ABI in <hbgpu.h>, so calibrate / run_hybrid
// (proj/src/scheduler.cpp), run_ea (proj/src/ea.cpp) and run_sweep via
// SweepHooks::make_accel (proj/include/hetbench/sweep.hpp:35-41) drive the
// GPU exactly as they drive synthetic_executor today.
//
// Error mapping (executor.cpp:60-65,121-128; scheduler.cpp:40-49):
//   HB_INVALID_ARG      -> std::invalid_argument (validate_request text)
//   HB_BLOWUP_PARTIAL   -> hetbench::batch_failure(failed sorted by seed,
//                          completed in order), numerical_blowup messages
//                          rebuilt by hb_format_blowup
//   other               -> std::runtime_error (back-end dead to calibrate)
#pragma once

#include <hbgpu.h>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hetbench/executor.hpp"

namespace hbgpu {

static_assert(sizeof(hb_variant_result) == sizeof(hetbench::VariantResult),
              "hb_variant_result must mirror hetbench::VariantResult");

class gpu_executor : public hetbench::batch_executor {
public:
    // monitor: fill BatchResult::utilization_trace (hb_ctx_set_monitor: NVML
    // samples while the call runs + the call's kernel-busy share), as
    // cpu_executor(workers, monitor = true) fills its CPU trace
    // (executor.hpp:78-80); the sweep's accel_util_mean comes from it
    // (sweep.cpp:119).
    explicit gpu_executor(int device = 0, bool monitor = true) {
        if (hb_ctx_create(device, &ctx_) != HB_OK)
            throw std::runtime_error(std::string("gpu_executor: ") + hb_global_error());
        if (monitor && hb_ctx_set_monitor(ctx_, 1) != HB_OK) {
            hb_ctx_destroy(ctx_);
            throw std::runtime_error(std::string("gpu_executor: ") + hb_global_error());
        }
        monitor_ = monitor;
    }
    ~gpu_executor() override { hb_ctx_destroy(ctx_); }
    gpu_executor(const gpu_executor&) = delete;
    gpu_executor& operator=(const gpu_executor&) = delete;

    hetbench::BatchResult run(const hetbench::BatchRequest& request) override {
        hetbench::validate_request(request);
        const std::size_t n = request.seeds.size();
        hetbench::BatchResult out;
        out.results.resize(n);
        std::vector<std::uint64_t> fail(n, 0);
        double wall = 0.0;
        const hb_status st =
            hb_run_batch(ctx_, static_cast<int>(request.kind), request.seeds.data(), n, request.steps,
                         reinterpret_cast<hb_variant_result*>(out.results.data()), fail.data(), &wall);
        if (st == HB_INVALID_ARG) throw std::invalid_argument(hb_last_error(ctx_));
        if (st == HB_BLOWUP_PARTIAL) {
            std::vector<std::pair<std::uint64_t, std::string>> failed;
            std::vector<hetbench::VariantResult> completed;
            for (std::size_t i = 0; i < n; ++i) {
                if (fail[i]) {
                    char buf[256];
                    hb_format_blowup(request.seeds[i], fail[i], hetbench::kSimDt, buf, sizeof buf);
                    failed.emplace_back(request.seeds[i], buf);
                } else {
                    completed.push_back(out.results[i]);
                }
            }
            std::sort(failed.begin(), failed.end());
            throw hetbench::batch_failure(std::move(failed), std::move(completed));
        }
        if (st != HB_OK) throw std::runtime_error(std::string("gpu_executor: ") + hb_last_error(ctx_));
        out.wall_time_s = wall;
        if (monitor_) {
            std::size_t count = 0;
            hb_last_utilization(ctx_, nullptr, 0, &count);
            std::vector<hb_util_sample> tr(count);
            hb_last_utilization(ctx_, tr.data(), tr.size(), &count);
            for (const hb_util_sample& u : tr) out.utilization_trace.push_back({u.t, u.accel_percent});
        }
        return out;
    }

    std::string name() const override { return "accel"; }
    hb_ctx* context() { return ctx_; }

    // Start-up reservation (hb_ctx_reserve): buffers sized and the kernel
    // loaded for batches of up to n variants of `kind`, so the first timed
    // run() — e.g. calibrate's single probe (scheduler.cpp:30-56) — is warm.
    void reserve(hetbench::ModelKind kind, std::size_t n) {
        if (hb_ctx_reserve(ctx_, static_cast<int>(kind), n) != HB_OK)
            throw std::runtime_error(std::string("gpu_executor: ") + hb_last_error(ctx_));
    }

private:
    hb_ctx* ctx_ = nullptr;
    bool monitor_ = true;
};

}  // namespace hbgpu
