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

    // Start-up reservation through the adapter (hb_ctx_reserve): a fresh
    // executor reserved for the probe size serves calibrate's single probe
    // warm, with results identical to an unreserved executor's.
    {
        std::vector<std::uint64_t> seeds(65536);
        std::iota(seeds.begin(), seeds.end(), std::uint64_t{0});
        BatchRequest req{ModelKind::ArmWithRope, seeds, 50};
        hbgpu::gpu_executor cold(0, /*monitor=*/false), warm(0, /*monitor=*/false);
        warm.reserve(ModelKind::ArmWithRope, seeds.size());
        const BatchResult a = cold.run(req), b = warm.run(req), c = warm.run(req);
        std::printf("  first call: unreserved %.3f ms, reserved %.3f ms (warm repeat %.3f ms)\n",
                    1e3 * a.wall_time_s, 1e3 * b.wall_time_s, 1e3 * c.wall_time_s);
        check(a.results == b.results && b.results == c.results && b.wall_time_s < a.wall_time_s,
              "reserve_first_call_warm_and_identical");
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
    // batch_failure mapping (executor.cpp:20-28,121-128): a variant reported
    // as blown up by the backend (hb_ctx_inject_fault, the test seam standing
    // in for a crafted state) surfaces as the reference's batch_failure with
    // the numerical_blowup text, and the rest of the batch completes.
    {
        std::vector<std::uint64_t> seeds(4096);
        std::iota(seeds.begin(), seeds.end(), std::uint64_t{0});
        const std::uint64_t bad = 3001;
        BatchRequest r{ModelKind::BoxAndBall, seeds, 300};
        const BatchResult want = cpu.run(r);
        hb_ctx_inject_fault(gpu.context(), HB_FAULT_BLOWUP, bad);
        bool ok = false;
        std::string detail = "no batch_failure";
        try {
            gpu.run(r);
        } catch (const batch_failure& e) {
            std::vector<VariantResult> rest;
            for (const VariantResult& v : want.results)
                if (v.seed != bad) rest.push_back(v);
            const std::string msg = "coordinate left the stable regime at t=0.002000 (seed 3001)";
            ok = e.failed().size() == 1 && e.failed()[0].first == bad && e.failed()[0].second == msg &&
                 e.completed() == rest &&
                 std::string(e.what()) == "batch failed for seed 3001: " + msg;
            detail = e.what();
        }
        check(ok, "batch_failure_mapping", detail);

        // run_hybrid (scheduler.cpp:162-183): the accelerator share throws
        // batch_failure, is re-dispatched to the CPU, the result is degraded
        // and the merge is the all-CPU result.
        const AllocationPlan plan = plan_allocation(CalibrationProfile{ModelKind::BoxAndBall, 300, 64, 1.0, 0.01,
                                                                       0.01, true, true},
                                                    seeds.size());
        const HybridResult hr = run_hybrid(plan, r, cpu, gpu, 0.0, ExecMode::Emulated);
        check(hr.degraded && hr.merged == want.results && plan.n_accel > 0, "run_hybrid_redispatch_on_blowup");

        // a dead device (HB_FAULT_DEVICE -> std::runtime_error): calibrate
        // flags the accelerator failed and the plan gives it nothing
        // (scheduler.cpp:40-49,70-72)
        hb_ctx_inject_fault(gpu.context(), HB_FAULT_DEVICE, 0);
        const CalibrationProfile p = calibrate(ModelKind::BoxAndBall, 300, 256, cpu, gpu);
        const AllocationPlan dead = plan_allocation(p, seeds.size());
        check(p.cpu_ok && !p.accel_ok && dead.n_accel == 0 && dead.n_cpu == seeds.size(),
              "calibrate_marks_dead_device");
        hb_ctx_inject_fault(gpu.context(), HB_FAULT_NONE, 0);
        check(gpu.run(r).results == want.results, "fault_reset");
    }
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
