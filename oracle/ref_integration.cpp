// ref_integration.cpp — TEST INFRASTRUCTURE ONLY.
//
// The drop-in demonstration: the UNMODIFIED reference library (its own
// calibrate / plan_allocation / run_hybrid / run_ea / cpu_executor, compiled
// from /root/reference/proj/src) driving the B200 backend through the
// reference-side adapter include/hbgpu/hetbench_gpu_executor.hpp.  Built by
// `make -C oracle integration` into oracle/_ref/ref_integration (travels to
// the GPU box prebuilt); run by tests/test_gpu_integration.py.
//
// Each check prints "PASS <name>" or "FAIL <name>: <detail>"; exit code =
// number of failures.
#include <cstdio>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "hbgpu/hetbench_gpu_executor.hpp"
#include "hetbench/ea.hpp"
#include "hetbench/rng.hpp"
#include "hetbench/scheduler.hpp"

using namespace hetbench;

static int g_fail = 0;
static void check(bool ok, const char* name, const std::string& detail = "") {
    if (ok) {
        std::printf("PASS %s\n", name);
    } else {
        std::printf("FAIL %s: %s\n", name, detail.c_str());
        ++g_fail;
    }
    std::fflush(stdout);
}

int main() {
    hbgpu::gpu_executor gpu(0);
    cpu_executor cpu(0, /*monitor=*/false);

    // C1 (acceptance.cpp:200-218): 200 (model, steps) cells, identical results.
    {
        const ModelKind kinds[] = {ModelKind::Box, ModelKind::BoxAndBall, ModelKind::ArmWithRope,
                                   ModelKind::Humanoid};
        const std::uint64_t steps_grid[] = {10, 100, 1000};
        std::map<std::pair<int, std::uint64_t>, std::vector<std::uint64_t>> groups;
        for (std::uint64_t i = 0; i < 200; ++i)
            groups[{static_cast<int>(kinds[i % 4]), steps_grid[(i / 4) % 3]}].push_back(rng::at(0xACC1, i));
        bool ok = true;
        std::size_t pairs = 0;
        for (const auto& [key, seeds] : groups) {
            BatchRequest r{static_cast<ModelKind>(key.first), seeds, key.second};
            const BatchResult a = cpu.run(r), b = gpu.run(r);
            ok = ok && a.results == b.results;
            pairs += seeds.size();
        }
        check(ok && pairs == 200, "c1_results_identical_200_pairs");
    }

    // executor contract (executor.cpp:183-198) at batch sizes that fill the GPU.
    for (ModelKind k : kAllModels) {
        std::vector<std::uint64_t> seeds(k == ModelKind::Humanoid ? 2048 : 8192);
        std::iota(seeds.begin(), seeds.end(), std::uint64_t{0});
        BatchRequest r{k, seeds, 200};
        const bool ok = cpu.run(r).results == gpu.run(r).results;
        check(ok, (std::string("contract_") + to_string(k)).c_str());
    }

    // request validation (executor.cpp:60-65)
    {
        bool threw = false;
        try {
            gpu.run(BatchRequest{ModelKind::Box, {}, 10});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        check(threw, "empty_request_invalid_argument");
    }

    // The paper's splitter on real back-ends: calibrate -> plan -> run_hybrid
    // (Emulated: both shares race on the real clock), merge == sequential.
    {
        const std::uint64_t steps = 1000;
        const CalibrationProfile p = calibrate(ModelKind::BoxAndBall, steps, 4096, cpu, gpu);
        std::vector<std::uint64_t> seeds(16384);
        std::iota(seeds.begin(), seeds.end(), std::uint64_t{0});
        BatchRequest req{ModelKind::BoxAndBall, seeds, steps};
        const AllocationPlan plan = plan_allocation(p, seeds.size());
        const HybridResult hr = run_hybrid(plan, req, cpu, gpu, 0.0, ExecMode::Emulated);
        const BatchResult ref = gpu.run(req);
        std::printf("  calibration: t_cpu=%.6f s t_accel=%.6f s ratio=%.6g\n", p.t_cpu_s, p.t_accel_s,
                    p.ratio_accel_over_cpu);
        std::printf("  plan: %s (accel_fraction=%.6f)\n", format_plan(plan).c_str(), plan.accel_fraction);
        std::printf("  wall_combined=%.6f s cpu_part=%.6f s accel_part=%.6f s\n", hr.wall_combined_s,
                    hr.t_cpu_part_s, hr.t_accel_part_s);
        check(p.cpu_ok && p.accel_ok && hr.merged == ref.results && !hr.degraded,
              "calibrate_plan_run_hybrid_merge");
    }

    // run_ea (ea.cpp:33-105) over the GPU executor == over cpu_executor.
    {
        const EaResult a = run_ea(ModelKind::BoxAndBall, 256, 3, 100, cpu, 11);
        const EaResult b = run_ea(ModelKind::BoxAndBall, 256, 3, 100, gpu, 11);
        check(a.population.genomes == b.population.genomes &&
                  a.population.fitnesses == b.population.fitnesses && a.best_fitness == b.best_fitness,
              "run_ea_box_and_ball_identical");
        const EaResult c = run_ea(ModelKind::Humanoid, 64, 2, 50, cpu, 3);
        const EaResult d = run_ea(ModelKind::Humanoid, 64, 2, 50, gpu, 3);
        check(c.population.genomes == d.population.genomes &&
                  c.population.fitnesses == d.population.fitnesses,
              "run_ea_humanoid_identical");
        std::printf("  run_ea over gpu_executor: evaluation_fraction=%.3f\n", b.profile.evaluation_fraction());
    }
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
