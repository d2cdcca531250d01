// ref_sweep.cpp — the paper's sweeps through the reference's OWN harness with
// the B200 in the accelerator slot (measurement infrastructure, not product).
//
// The unmodified reference run_sweep (proj/src/sweep.cpp:61-164) with
// SweepHooks::make_accel (proj/include/hetbench/sweep.hpp:35-41) returning
// hbgpu::gpu_executor (include/hbgpu/hetbench_gpu_executor.hpp, monitor on:
// accel_util_mean of every accel row comes from its utilization_trace,
// sweep.cpp:119), the reference cpu_executor as "cpu", the reference's
// calibrate / plan_allocation / run_hybrid for "hybrid" cells, its CSV /
// JSONL records and its figures (figures.cpp: <model>_wall_vs_n.svg,
// <model>_accel_wall_util.svg, <model>_combined_overlay.svg,
// <model>_wall_vs_steps.svg + .csv sidecars).  Afterwards the saturation
// knee of every model's accel and cpu series by the reference's
// detect_saturation_knee (monitor.cpp:184-203), as its `knee` command does
// (tools/hetbench_main.cpp:236-262), into <out>/knees.txt.
//
// Built by `make -C oracle sweep` from the reference sources in place into
// oracle/_ref/ref_sweep (git-ignored; travels to the GPU box prebuilt).
//   usage: ref_sweep <config.toml> <output_dir> [device]
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "hbgpu/hetbench_gpu_executor.hpp"
#include "hetbench/config.hpp"
#include "hetbench/monitor.hpp"
#include "hetbench/sweep.hpp"

using namespace hetbench;

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <config.toml> <output_dir> [device]\n", argv[0]);
        return 1;
    }
    const int device = argc > 3 ? std::atoi(argv[3]) : 0;
    try {
        SweepConfig cfg = load_sweep_config(argv[1]);
        cfg.output_dir = argv[2];
        validate_config(cfg);
        SweepHooks hooks;
        // start-up: every model's buffers sized for its largest variant count
        // and its kernels loaded (hb_ctx_reserve), so the sweep's first rows
        // and calibrate's single probe time warm calls, as a long-running
        // accelerator service would serve them
        hooks.make_accel = [device](const SweepConfig& c) -> std::unique_ptr<batch_executor> {
            auto ex = std::make_unique<hbgpu::gpu_executor>(device, /*monitor=*/true);
            for (const auto& [model, counts] : c.variants_per_model) {
                std::uint64_t mx = 0;
                for (std::uint64_t v : counts) mx = std::max(mx, v);
                if (c.hybrid_probe_n > mx) mx = c.hybrid_probe_n;
                ex->reserve(model, mx);
            }
            return ex;
        };
        const std::uint64_t total = expected_row_count(cfg);
        std::uint64_t seen = 0;
        hooks.on_record = [&](const RunRecord& r) {
            ++seen;
            std::printf("[%llu/%llu] %s wall=%s s util=%s%s\n", static_cast<unsigned long long>(seen),
                        static_cast<unsigned long long>(total), record_key(r).c_str(), format_g6(r.wall_s).c_str(),
                        format_g6(r.strategy == Strategy::CpuOnly ? r.cpu_util_mean : r.accel_util_mean).c_str(),
                        r.error() ? " (error)" : (r.degraded ? " (degraded)" : ""));
            std::fflush(stdout);
        };
        const SweepOutcome out = run_sweep(cfg, false, hooks);
        std::printf("rows_written=%llu error_rows=%llu degraded_rows=%llu\n",
                    static_cast<unsigned long long>(out.rows_written),
                    static_cast<unsigned long long>(out.error_rows),
                    static_cast<unsigned long long>(out.degraded_rows));
        for (const auto& f : out.figure_files) std::printf("figure: %s\n", f.string().c_str());

        std::ofstream knees(cfg.output_dir / "knees.txt");
        for (ModelKind kind : cfg.models)
            for (Strategy strat : {Strategy::AccelOnly, Strategy::CpuOnly}) {
                std::uint64_t steps = 0;
                for (const RunRecord& r : out.records)
                    if (r.model == kind && r.strategy == strat && !r.error()) steps = std::max(steps, r.steps);
                std::map<std::uint64_t, std::vector<double>> walls;
                for (const RunRecord& r : out.records)
                    if (r.model == kind && r.strategy == strat && !r.error() && r.steps == steps)
                        walls[r.n_variants].push_back(r.wall_s);
                if (walls.size() < 3) continue;
                std::vector<KneePoint> points;
                for (const auto& [n, w] : walls) points.push_back({n, summarize(w).mean});
                const KneeResult kr = detect_saturation_knee(points, 0.05);
                const char* regime = kr.regime == KneeRegime::Knee      ? "knee"
                                     : kr.regime == KneeRegime::AllFlat ? "all_flat"
                                                                        : "all_linear";
                char line[256];
                std::snprintf(line, sizeof line, "knee: n=%llu regime=%s model=%s strategy=%s steps=%llu\n",
                              static_cast<unsigned long long>(kr.n), regime, to_string(kind), to_string(strat).c_str(),
                              static_cast<unsigned long long>(steps));
                std::fputs(line, stdout);
                knees << line;
            }
        return out.error_rows > 0 ? 3 : 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
