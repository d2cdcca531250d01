// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, compiled in
// place from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libhetbench_ref.so (git-ignored; it travels to the GPU box as a
// prebuilt file).  Used (a) to pin the C restatement oracle/hb_oracle.c,
// (b) to generate tests/golden/, and (c) as bench.py's reference arm /
// cpu_baseline ("kind": "reference"): the reference's own cpu_executor
// (proj/src/executor.cpp:79-135) timed on the host cores.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "hetbench/ea.hpp"
#include "hetbench/executor.hpp"
#include "hetbench/monitor.hpp"
#include "hetbench/rng.hpp"
#include "hetbench/scheduler.hpp"
#include "hetbench/simkernel.hpp"

using namespace hetbench;

namespace {
void copy_msg(const std::string& s, char* buf, std::size_t cap) {
    if (!buf || cap == 0) return;
    std::size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
}
}  // namespace

extern "C" {

static_assert(sizeof(VariantResult) == 32, "VariantResult layout");

unsigned hbref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// simulate (simkernel.cpp:187-203). 0 ok, 1 numerical_blowup, 2 other error.
int hbref_simulate(int kind, std::uint64_t seed, std::uint64_t steps, VariantResult* out,
                   char* msg, std::size_t cap) {
    try {
        *out = simulate(static_cast<ModelKind>(kind), seed, steps);
        return 0;
    } catch (const numerical_blowup& e) {
        copy_msg(e.what(), msg, cap);
        return 1;
    } catch (const std::exception& e) {
        copy_msg(e.what(), msg, cap);
        return 2;
    }
}

// build_model (simkernel.cpp:59-120): AoS positions / velocities, rest lengths.
int hbref_build_model(int kind, std::uint64_t seed, double* pos, double* vel, double* rest,
                      std::uint64_t* ca, std::uint64_t* cb, double* stiff) {
    WorldState w = build_model(static_cast<ModelKind>(kind), seed);
    for (std::size_t i = 0; i < w.positions.size(); ++i) {
        pos[3 * i] = w.positions[i].x; pos[3 * i + 1] = w.positions[i].y; pos[3 * i + 2] = w.positions[i].z;
        vel[3 * i] = w.velocities[i].x; vel[3 * i + 1] = w.velocities[i].y; vel[3 * i + 2] = w.velocities[i].z;
    }
    for (std::size_t k = 0; k < w.constraints.size(); ++k) {
        rest[k] = w.constraints[k].rest_length;
        if (ca) ca[k] = w.constraints[k].a;
        if (cb) cb[k] = w.constraints[k].b;
        if (stiff) stiff[k] = w.constraints[k].stiffness;
    }
    return static_cast<int>(w.constraints.size());
}

// build_model + `steps` x step(kSimDt), returning the full final state
// (for trajectory parity at intermediate horizons). 0 ok, 1 blow-up.
int hbref_trajectory(int kind, std::uint64_t seed, std::uint64_t steps, double* pos, double* vel,
                     double* time) {
    WorldState w = build_model(static_cast<ModelKind>(kind), seed);
    int rc = 0;
    try {
        for (std::uint64_t s = 0; s < steps; ++s) step(w, kSimDt);
    } catch (const numerical_blowup&) {
        rc = 1;
    }
    for (std::size_t i = 0; i < w.positions.size(); ++i) {
        pos[3 * i] = w.positions[i].x; pos[3 * i + 1] = w.positions[i].y; pos[3 * i + 2] = w.positions[i].z;
        vel[3 * i] = w.velocities[i].x; vel[3 * i + 1] = w.velocities[i].y; vel[3 * i + 2] = w.velocities[i].z;
    }
    *time = w.time;
    return rc;
}

// One reference step() on a caller-supplied state (known-answer tests,
// test_simkernel.cpp:106-126,182-186).  0 ok, 1 blow-up, 2 invalid dt.
int hbref_step_state(int kind, double* pos, double* vel, double dt, std::uint64_t seed_for_topology,
                     char* msg, std::size_t cap) {
    WorldState w = build_model(static_cast<ModelKind>(kind), seed_for_topology);
    for (std::size_t i = 0; i < w.positions.size(); ++i) {
        w.positions[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        w.velocities[i] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
    }
    int rc = 0;
    try {
        step(w, dt);
    } catch (const numerical_blowup& e) {
        copy_msg(e.what(), msg, cap);
        rc = 1;
    } catch (const std::invalid_argument& e) {
        copy_msg(e.what(), msg, cap);
        return 2;
    }
    for (std::size_t i = 0; i < w.positions.size(); ++i) {
        pos[3 * i] = w.positions[i].x; pos[3 * i + 1] = w.positions[i].y; pos[3 * i + 2] = w.positions[i].z;
        vel[3 * i] = w.velocities[i].x; vel[3 * i + 1] = w.velocities[i].y; vel[3 * i + 2] = w.velocities[i].z;
    }
    return rc;
}

std::uint64_t hbref_state_checksum(int kind, std::uint64_t seed) {
    return state_checksum(build_model(static_cast<ModelKind>(kind), seed));
}

// The reference CPU stepping loop: cpu_executor(workers, monitor=false).run
// (executor.cpp:79-135).  Returns 0 ok, 1 batch_failure (failed seeds
// written to failed_seeds, count to *n_failed, what() to msg), 2 other error.
int hbref_cpu_run(int kind, const std::uint64_t* seeds, std::size_t n, std::uint64_t steps,
                  unsigned workers, VariantResult* out, double* wall_time_s,
                  std::uint64_t* failed_seeds, std::size_t* n_failed, char* msg, std::size_t cap) {
    try {
        cpu_executor exec(workers, /*monitor=*/false);
        BatchRequest req{static_cast<ModelKind>(kind), {seeds, seeds + n}, steps};
        BatchResult r = exec.run(req);
        std::memcpy(out, r.results.data(), n * sizeof(VariantResult));
        if (wall_time_s) *wall_time_s = r.wall_time_s;
        if (n_failed) *n_failed = 0;
        return 0;
    } catch (const batch_failure& e) {
        copy_msg(e.what(), msg, cap);
        if (n_failed) *n_failed = e.failed().size();
        if (failed_seeds)
            for (std::size_t i = 0; i < e.failed().size(); ++i) failed_seeds[i] = e.failed()[i].first;
        return 1;
    } catch (const std::exception& e) {
        copy_msg(e.what(), msg, cap);
        return 2;
    }
}

// plan_allocation (scheduler.cpp:58-87).
int hbref_plan_allocation(double t_cpu, double t_accel, int cpu_ok, int accel_ok,
                          std::uint64_t n_total, AllocationPlan* out) {
    try {
        CalibrationProfile p;
        p.t_cpu_s = t_cpu;
        p.t_accel_s = t_accel;
        p.cpu_ok = cpu_ok != 0;
        p.accel_ok = accel_ok != 0;
        *out = plan_allocation(p, n_total);
        return 0;
    } catch (const std::exception&) {
        return 2;
    }
}

// run_ea (ea.cpp:33-105) over cpu_executor(workers, monitor=false).
int hbref_run_ea(int kind, std::size_t pop, std::uint64_t generations, std::uint64_t steps,
                 std::uint64_t seed, unsigned workers, std::uint64_t* genomes, double* fitness,
                 double* best) {
    try {
        cpu_executor exec(workers, /*monitor=*/false);
        EaResult r = run_ea(static_cast<ModelKind>(kind), pop, generations, steps, exec, seed);
        for (std::size_t i = 0; i < pop; ++i) {
            genomes[i] = r.population.genomes[i];
            fitness[i] = r.population.fitnesses[i];
        }
        if (best) *best = r.best_fitness;
        return 0;
    } catch (const std::exception&) {
        return 2;
    }
}

// detect_saturation_knee (monitor.cpp:184-203), reused unchanged for the
// measured B200 variant sweeps.
int hbref_detect_knee(const std::uint64_t* n, const double* wall, std::size_t count, double eps,
                      std::uint64_t* knee_n, int* regime) {
    try {
        std::vector<KneePoint> pts(count);
        for (std::size_t i = 0; i < count; ++i) pts[i] = {n[i], wall[i]};
        KneeResult k = detect_saturation_knee(pts, eps);
        *knee_n = k.n;
        *regime = static_cast<int>(k.regime);
        return 0;
    } catch (const std::exception&) {
        return 2;
    }
}

// Reference blow-up text after `s_before` normal steps followed by one step
// with body 0 kicked to v.z = 1e9 (test_simkernel.cpp:182-186 at a horizon):
// the numerical_blowup what() of step() (simkernel.cpp:165-169), time included.
int hbref_blowup_after(int kind, std::uint64_t seed, std::uint64_t s_before, char* msg,
                       std::size_t cap) {
    WorldState w = build_model(static_cast<ModelKind>(kind), seed);
    try {
        for (std::uint64_t s = 0; s < s_before; ++s) step(w, kSimDt);
        w.velocities[0].z = 1e9;
        step(w, kSimDt);
    } catch (const numerical_blowup& e) {
        copy_msg(e.what(), msg, cap);
        return 1;
    }
    return 0;
}

std::uint64_t hbref_rng_at(std::uint64_t key, std::uint64_t ctr) { return rng::at(key, ctr); }

}  // extern "C"
