/*
 * hb_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference `hetbench` hot path, used as the
 * parity checker for the CUDA product path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library; the product
 * (paper_2502_11129_b200/) never links or calls it.
 *
 * Parity pinning: this restatement is checked against
 *   (1) oracle/_ref/libhetbench_ref.so — the reference sources compiled in
 *       place from /root/reference/proj/src by oracle/Makefile, and
 *   (2) the committed golden vectors in tests/golden/ (generated from (1) by
 *       tests/golden/make_golden.py, including SURVEY.md Appendix A values).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Arithmetic is IEEE double in the reference's source
 * order; compile with -ffp-contract=off (the reference -O3 build has no FMA).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hb_oracle.h"

/* ---- rng: include/hetbench/rng.hpp:15-49 -------------------------------- */
uint64_t hbo_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

uint64_t hbo_rng_at(uint64_t key, uint64_t counter) {
    return hbo_mix64(hbo_mix64(key + 0x9E3779B97F4A7C15ull) ^
                     (counter * 0xD1B54A32D192ED03ull + 1));
}

double hbo_to_unit(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

typedef struct {
    uint64_t key, ctr;
} stream_t;

static double s_unit(stream_t* s) { return hbo_to_unit(hbo_rng_at(s->key, s->ctr++)); }
/* RngStream::next_range  rng.hpp:44 : lo + (hi - lo) * next_unit() */
static double s_range(stream_t* s, double lo, double hi) { return lo + (hi - lo) * s_unit(s); }

/* ---- topology: include/hetbench/simkernel.hpp:23-31, src/simkernel.cpp:95-118 */
int hbo_body_count(int kind) {
    switch (kind) {
        case HBO_BOX: return 1;
        case HBO_BOX_AND_BALL: return 2;
        case HBO_ARM_WITH_ROPE: return 12;
        case HBO_HUMANOID: return 32;
        case HBO_CPG_HINGE: return 9;
    }
    return 0;
}

int hbo_constraint_count(int kind) {
    switch (kind) {
        case HBO_BOX: return 0;
        case HBO_BOX_AND_BALL: return 1;
        case HBO_ARM_WITH_ROPE: return 11;
        case HBO_HUMANOID: return 46;
        case HBO_CPG_HINGE: return 12;
    }
    return 0;
}

static const double kStiffLink = 2.5e5; /* simkernel.cpp:13 */
static const double kSoftLink = 1.25e5; /* simkernel.cpp:14 */

/* Constraint list in reference order (add_chain simkernel.cpp:35-40 and the
 * switch at :95-118). */
static void topology(int kind, int* ca, int* cb, double* stiff) {
    int m = 0;
    switch (kind) {
        case HBO_BOX: break;
        case HBO_BOX_AND_BALL:
            ca[m] = 0; cb[m] = 1; stiff[m++] = kStiffLink;
            break;
        case HBO_ARM_WITH_ROPE:
            for (int i = 0; i < 5; ++i) { ca[m] = i; cb[m] = i + 1; stiff[m++] = kStiffLink; }
            for (int i = 5; i < 11; ++i) { ca[m] = i; cb[m] = i + 1; stiff[m++] = kSoftLink; }
            break;
        case HBO_HUMANOID:
            for (int i = 0; i < 15; ++i) { ca[m] = i; cb[m] = i + 1; stiff[m++] = kStiffLink; }
            for (int i = 16; i < 31; ++i) { ca[m] = i; cb[m] = i + 1; stiff[m++] = kStiffLink; }
            for (int i = 0; i < 16; ++i) { ca[m] = i; cb[m] = 16 + i; stiff[m++] = kStiffLink; }
            break;
        case HBO_CPG_HINGE:
            /* NOT IN THE REFERENCE — see cpg section below. */
            for (int l = 0; l < 4; ++l) {
                ca[m] = 0; cb[m] = 1 + 2 * l; stiff[m++] = kStiffLink;          /* core - hinge */
                ca[m] = 1 + 2 * l; cb[m] = 2 + 2 * l; stiff[m++] = kStiffLink;  /* hinge - tip */
            }
            for (int l = 0; l < 4; ++l) { ca[m] = 0; cb[m] = 2 + 2 * l; stiff[m++] = kSoftLink; }
            break;
    }
}

int hbo_topology(int kind, int* ca, int* cb, double* stiff) {
    if (kind < 0 || kind > 4) return -1;
    topology(kind, ca, cb, stiff);
    return hbo_constraint_count(kind);
}

static double dist3(const double* p, int a, int b) {
    /* Vec3::norm  vec3.hpp:22-23 : sqrt(x*x + y*y + z*z), left to right */
    const double dx = p[3 * b + 0] - p[3 * a + 0];
    const double dy = p[3 * b + 1] - p[3 * a + 1];
    const double dz = p[3 * b + 2] - p[3 * a + 2];
    return sqrt(dx * dx + dy * dy + dz * dz);
}

/* build_model  simkernel.cpp:59-120.  pos/vel: AoS [body][xyz]; rest: [m]. */
int hbo_cpg_build(uint64_t seed, double* pos, double* vel, double* rest, double* cpg);

int hbo_build_model(int kind, uint64_t seed, double* pos, double* vel, double* rest) {
    if (kind == HBO_CPG_HINGE) {
        double cpg[16];
        return hbo_cpg_build(seed, pos, vel, rest, cpg);
    }
    if (kind < 0 || kind > 3) return -1;
    stream_t rs = {seed, 0};
    const double drop_height = s_range(&rs, 0.5, 2.0);
    const double lx = s_range(&rs, -1.0, 1.0);
    const double ly = s_range(&rs, -1.0, 1.0);
    const double heading = s_range(&rs, 0.0, 2.0 * 3.14159265358979323846);

    const int n = hbo_body_count(kind);
    const int twin = kind == HBO_HUMANOID;
    const double spacing = twin ? 0.12 : 0.25;
    for (int i = 0; i < n; ++i) {
        const int j = twin ? i % 16 : i;
        const double a = heading + 0.15 * (double)j;
        const double c = cos(a), s = sin(a);
        double x = spacing * (double)j * c;
        double y = spacing * (double)j * s;
        double z = drop_height + 0.05 * (double)j;
        if (twin && i >= 16) {
            x -= spacing * s;
            y += spacing * c;
        }
        x += 1e-3 * s_range(&rs, -1.0, 1.0);
        y += 1e-3 * s_range(&rs, -1.0, 1.0);
        z += 1e-3 * s_unit(&rs);
        pos[3 * i + 0] = x;
        pos[3 * i + 1] = y;
        pos[3 * i + 2] = z;
        vel[3 * i + 0] = lx;
        vel[3 * i + 1] = ly;
        vel[3 * i + 2] = 0.0;
    }
    int ca[46], cb[46];
    double st[46];
    topology(kind, ca, cb, st);
    const int m = hbo_constraint_count(kind);
    for (int k = 0; k < m; ++k) rest[k] = dist3(pos, ca[k], cb[k]);
    return 0;
}

static int coordinate_ok(const double* v) {
    /* simkernel.cpp:28-32 */
    for (int c = 0; c < 3; ++c)
        if (!isfinite(v[c]) || !(fabs(v[c]) <= 1e6)) return 0;
    return 1;
}

/* step  simkernel.cpp:122-170.  Returns 0 ok, 1 numerical blow-up, -1 bad dt.
 * `time` is advanced exactly as WorldState::time (:163). */
int hbo_step(int kind, double* pos, double* vel, const double* rest, double dt, double* time) {
    if (!(dt > 0.0)) return -1;
    const int n = hbo_body_count(kind);
    const int m = hbo_constraint_count(kind);
    int ca[46], cb[46];
    double st[46];
    topology(kind, ca, cb, st);

    const double damp = 1.0 - 0.8 * dt; /* :126, damping = 0.8 (:62) */
    for (int i = 0; i < n; ++i) {
        vel[3 * i + 2] -= 9.81 * dt;
        vel[3 * i + 0] *= damp;
        vel[3 * i + 1] *= damp;
        vel[3 * i + 2] *= damp;
    }
    double pred[96];
    for (int i = 0; i < 3 * n; ++i) pred[i] = pos[i] + vel[i] * dt; /* :134-136 */

    for (int it = 0; it < 8; ++it) { /* :140-152 */
        for (int k = 0; k < m; ++k) {
            const int a = ca[k], b = cb[k];
            const double dx = pred[3 * b + 0] - pred[3 * a + 0];
            const double dy = pred[3 * b + 1] - pred[3 * a + 1];
            const double dz = pred[3 * b + 2] - pred[3 * a + 2];
            const double dist = sqrt(dx * dx + dy * dy + dz * dz);
            if (dist < 1e-12) continue;
            const double kx = st[k] * dt * dt;
            const double kk = (kx < 1.0) ? kx : 1.0; /* std::min(1.0, kx) */
            const double corr = 0.5 * kk * (dist - rest[k]) / dist;
            pred[3 * a + 0] += dx * corr;
            pred[3 * a + 1] += dy * corr;
            pred[3 * a + 2] += dz * corr;
            pred[3 * b + 0] -= dx * corr;
            pred[3 * b + 1] -= dy * corr;
            pred[3 * b + 2] -= dz * corr;
        }
        for (int i = 0; i < n; ++i)
            if (pred[3 * i + 2] < 0.0) pred[3 * i + 2] = 0.0;
    }

    const double inv_dt = 1.0 / dt; /* :156-162 */
    for (int i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c) {
            vel[3 * i + c] = (pred[3 * i + c] - pos[3 * i + c]) * inv_dt;
            pos[3 * i + c] = pred[3 * i + c];
        }
        if (pos[3 * i + 2] <= 0.0 && vel[3 * i + 2] < 0.0) vel[3 * i + 2] = 0.0;
    }
    *time += dt;
    for (int i = 0; i < n; ++i) /* :165-169 */
        if (!coordinate_ok(pos + 3 * i) || !coordinate_ok(vel + 3 * i)) return 1;
    return 0;
}

/* state_checksum / fnv_absorb  simkernel.cpp:16-26,172-185 */
static uint64_t fnv_absorb(uint64_t h, double value) {
    uint64_t bits;
    memcpy(&bits, &value, sizeof bits);
    for (int i = 0; i < 8; ++i) {
        h ^= (bits >> (8 * i)) & 0xffu;
        h *= 0x100000001b3ull;
    }
    return h;
}

uint64_t hbo_checksum(int n, const double* pos, const double* vel) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int i = 0; i < 3 * n; ++i) h = fnv_absorb(h, pos[i]);
    for (int i = 0; i < 3 * n; ++i) h = fnv_absorb(h, vel[i]);
    return h;
}

/* simulate  simkernel.cpp:187-203.  Returns 0 ok, 1 blow-up (fail_step =
 * number of steps executed incl. the failing one), -1 invalid argument. */
int hbo_cpg_simulate(uint64_t seed, uint64_t steps, hbo_result* out, uint64_t* fail_step);

int hbo_simulate(int kind, uint64_t seed, uint64_t steps, hbo_result* out, uint64_t* fail_step) {
    if (kind == HBO_CPG_HINGE) return hbo_cpg_simulate(seed, steps, out, fail_step);
    if (steps < 1 || kind < 0 || kind > 3) return -1;
    double pos[96], vel[96], rest[46];
    hbo_build_model(kind, seed, pos, vel, rest);
    const int n = hbo_body_count(kind);
    const double sx = pos[0], sy = pos[1];
    double time = 0.0;
    for (uint64_t s = 0; s < steps; ++s) {
        if (hbo_step(kind, pos, vel, rest, 0.002, &time) == 1) {
            if (fail_step) *fail_step = s + 1;
            return 1;
        }
    }
    const double dx = pos[0] - sx, dy = pos[1] - sy;
    out->seed = seed;
    out->fitness = sqrt(dx * dx + dy * dy);
    out->checksum = hbo_checksum(n, pos, vel);
    out->steps_executed = steps;
    if (fail_step) *fail_step = 0;
    return 0;
}

/* Time after `steps` additions of dt starting at 0.0 (WorldState::time,
 * simkernel.cpp:163) — used to rebuild numerical_blowup messages. */
double hbo_time_after(uint64_t steps, double dt) {
    double t = 0.0;
    for (uint64_t s = 0; s < steps; ++s) t += dt;
    return t;
}

/* Message of simulate's re-thrown numerical_blowup (simkernel.cpp:167-168,194):
 * "coordinate left the stable regime at t=<to_string(time)> (seed <seed>)". */
int hbo_blowup_message(uint64_t seed, uint64_t fail_step, double dt, char* buf, size_t cap) {
    return snprintf(buf, cap, "coordinate left the stable regime at t=%f (seed %llu)",
                    hbo_time_after(fail_step, dt), (unsigned long long)seed);
}

/* ---- batch (checker helper; contiguous chunks like executor.cpp:93-113) -- */
typedef struct {
    int kind;
    const uint64_t* seeds;
    size_t begin, end;
    uint64_t steps;
    hbo_result* out;
    uint64_t* fail;
} job_t;

static void* run_job(void* p) {
    job_t* j = (job_t*)p;
    for (size_t i = j->begin; i < j->end; ++i) {
        uint64_t fs = 0;
        hbo_result r = {0, 0.0, 0, 0};
        hbo_simulate(j->kind, j->seeds[i], j->steps, &r, &fs);
        j->out[i] = r;
        if (j->fail) j->fail[i] = fs;
    }
    return NULL;
}

int hbo_simulate_batch(int kind, const uint64_t* seeds, size_t n, uint64_t steps, int threads,
                       hbo_result* out, uint64_t* fail_step) {
    if (steps < 1 || n == 0 || kind < 0 || kind > 4) return -1;
    if (threads < 1) threads = 1;
    if ((size_t)threads > n) threads = (int)n;
    pthread_t tid[256];
    job_t jobs[256];
    if (threads > 256) threads = 256;
    const size_t chunk = n / threads, extra = n % threads;
    size_t begin = 0;
    for (int w = 0; w < threads; ++w) {
        const size_t end = begin + chunk + ((size_t)w < extra ? 1 : 0);
        jobs[w] = (job_t){kind, seeds, begin, end, steps, out, fail_step};
        begin = end;
        if (threads == 1) run_job(&jobs[w]);
        else pthread_create(&tid[w], NULL, run_job, &jobs[w]);
    }
    if (threads > 1)
        for (int w = 0; w < threads; ++w) pthread_join(tid[w], NULL);
    return 0;
}

/* ---- splitter: scheduler.cpp:58-87 --------------------------------------- */
int hbo_plan_allocation(double t_cpu, double t_accel, int cpu_ok, int accel_ok, uint64_t n_total,
                        hbo_plan* plan) {
    if (n_total < 1) return -1;
    memset(plan, 0, sizeof *plan);
    plan->n_total = n_total;
    if (!accel_ok) {
        plan->n_accel = 0;
    } else if (!cpu_ok) {
        plan->n_accel = n_total;
        plan->requested_accel_fraction = 1.0;
    } else {
        const double f = t_cpu / (t_cpu + t_accel);
        plan->requested_accel_fraction = f;
        uint64_t na = (uint64_t)llround(f * (double)n_total);
        if (na > n_total) na = n_total;
        const double thr = 1.0 / (2.0 * (double)n_total);
        if (na == 0 && f >= thr) na = 1;
        if (na == n_total && (1.0 - f) >= thr) na = n_total - 1;
        plan->n_accel = na;
    }
    plan->n_cpu = n_total - plan->n_accel;
    plan->accel_fraction = (double)plan->n_accel / (double)n_total;
    return 0;
}

/* ---- EA: ea.cpp:33-105 (selection = stable sort by fitness descending) -- */
static const double* g_sort_fit;
static int cmp_desc_stable(const void* a, const void* b) {
    const size_t ia = *(const size_t*)a, ib = *(const size_t*)b;
    const double fa = g_sort_fit[ia], fb = g_sort_fit[ib];
    if (fa > fb) return -1;
    if (fb > fa) return 1;
    return (ia < ib) ? -1 : (ia > ib); /* ties keep input order (stable) */
}

/* Order of indices std::stable_sort(order, fitness[a] > fitness[b]) yields
 * (ea.cpp:60-66).  Not thread-safe (qsort comparator global). */
void hbo_stable_order_desc(const double* fitness, size_t n, size_t* order) {
    for (size_t i = 0; i < n; ++i) order[i] = i;
    g_sort_fit = fitness;
    qsort(order, n, sizeof(size_t), cmp_desc_stable);
}

uint64_t hbo_init_genome(uint64_t seed, uint64_t i) { return hbo_rng_at(seed ^ 0x8F5D4C3B2A190807ull, i); }
uint64_t hbo_child_genome(uint64_t parent, uint64_t g, uint64_t i) {
    return hbo_rng_at(parent ^ 0x243F6A8885A308D3ull, (g << 32) + i);
}

/* Full run_ea with the oracle batch evaluator; genomes/fitness out = final
 * population (parents ++ offspring).  Returns 0 ok, 1 blow-up, -1 args. */
int hbo_run_ea(int kind, size_t pop, uint64_t generations, uint64_t steps, uint64_t seed,
               int threads, uint64_t* genomes, double* fitness) {
    if (pop < 2 || pop % 2 || generations < 1) return -1;
    const size_t mu = pop / 2;
    hbo_result* res = (hbo_result*)malloc(sizeof(hbo_result) * pop);
    uint64_t* fail = (uint64_t*)malloc(sizeof(uint64_t) * pop);
    size_t* order = (size_t*)malloc(sizeof(size_t) * pop);
    uint64_t* par = (uint64_t*)malloc(sizeof(uint64_t) * mu);
    double* pfit = (double*)malloc(sizeof(double) * mu);
    int rc = 0;
    for (size_t i = 0; i < pop; ++i) genomes[i] = hbo_init_genome(seed, i);
    hbo_simulate_batch(kind, genomes, pop, steps, threads, res, fail);
    for (size_t i = 0; i < pop; ++i) {
        if (fail[i]) rc = 1;
        fitness[i] = res[i].fitness;
    }
    for (uint64_t g = 1; g <= generations && rc == 0; ++g) {
        hbo_stable_order_desc(fitness, pop, order);
        for (size_t i = 0; i < mu; ++i) {
            par[i] = genomes[order[i]];
            pfit[i] = fitness[order[i]];
        }
        for (size_t i = 0; i < mu; ++i) genomes[mu + i] = hbo_child_genome(par[i], g, i);
        hbo_simulate_batch(kind, genomes + mu, mu, steps, threads, res, fail);
        for (size_t i = 0; i < mu; ++i) {
            if (fail[i]) rc = 1;
            genomes[i] = par[i];
            fitness[i] = pfit[i];
            fitness[mu + i] = res[i].fitness;
        }
    }
    free(res); free(fail); free(order); free(par); free(pfit);
    return rc;
}

/* ===========================================================================
 * CPG / hinge modular robot (kind 4) — NOT IN THE REFERENCE.
 *
 * BASELINE config 3 names a "Revolve2-style modular robot with hinge joints +
 * CPG controller"; the reference has none ("joint torque actuation,
 * controller evolution" are non-goals).  This is its
 * definition, in simkernel style; the CUDA path is
 * checked against THIS restatement, so its parity is unpinned by the
 * reference.
 *
 * Bodies (9): core 0; limb l = 0..3 at angle a_l = heading + l*RN(pi/2):
 *   hinge 1+2l at 0.25 m along a_l, 0.10 m above the core;
 *   tip   2+2l at 0.50 m along a_l, 0.05 m above the core;
 *   jitter and launch velocity exactly as build_model (simkernel.cpp:59-92).
 * Constraints (12, list order): core-hinge, hinge-tip (stiff) per limb,
 *   then the four actuated core-tip "hinges" (soft) whose rest length is
 *   L0_l * (1 + 0.2 * u_l), L0_l the initial distance.
 * CPG per joint l: state (x_l, y_l), parameters omega_l = 2pi * U[0.5, 2),
 *   c_l = U[-0.5, 0.5) (coupling to joint (l+1) & 3), x_l(0) = U[-0.1, 0.1),
 *   y_l(0) = 0, drawn from RngStream(seed ^ kCpgKey) in that order.
 * Step: CPG first (symplectic Euler on the old state),
 *     nx_l = x_l + dt * (omega_l * y_l + c_l * x_{(l+1)&3})
 *     y_l  = y_l - dt * (omega_l * nx_l);  x_l = nx_l
 *     u_l  = clamp(x_l, -1, 1)
 *   then the reference step() with the updated rest lengths.
 * Checksum: FNV-1a over positions, velocities, then x[4], y[4].
 * Known answer: omega = c = x(0) = 0 keeps every rest length at L0 exactly,
 * i.e. the passive robot.
 * ======================================================================== */
static const uint64_t kCpgKey = 0xC0FFEE5EEDC0DE5Full;

int hbo_cpg_build(uint64_t seed, double* pos, double* vel, double* rest, double* cpg) {
    stream_t rs = {seed, 0};
    const double drop_height = s_range(&rs, 0.5, 2.0);
    const double lx = s_range(&rs, -1.0, 1.0);
    const double ly = s_range(&rs, -1.0, 1.0);
    const double heading = s_range(&rs, 0.0, 2.0 * 3.14159265358979323846);
    for (int i = 0; i < 9; ++i) {
        double x, y, z;
        if (i == 0) {
            x = 0.0; y = 0.0; z = drop_height;
        } else {
            const int l = (i - 1) / 2;
            const int tip = (i - 1) % 2;
            const double a = heading + 1.5707963267948966 * (double)l;
            const double r = tip ? 0.50 : 0.25;
            x = r * cos(a);
            y = r * sin(a);
            z = drop_height + (tip ? 0.05 : 0.10);
        }
        x += 1e-3 * s_range(&rs, -1.0, 1.0);
        y += 1e-3 * s_range(&rs, -1.0, 1.0);
        z += 1e-3 * s_unit(&rs);
        pos[3 * i + 0] = x; pos[3 * i + 1] = y; pos[3 * i + 2] = z;
        vel[3 * i + 0] = lx; vel[3 * i + 1] = ly; vel[3 * i + 2] = 0.0;
    }
    int ca[12], cb[12];
    double st[12];
    topology(HBO_CPG_HINGE, ca, cb, st);
    for (int k = 0; k < 12; ++k) rest[k] = dist3(pos, ca[k], cb[k]);
    stream_t cs = {seed ^ kCpgKey, 0};
    for (int l = 0; l < 4; ++l) cpg[8 + l] = (2.0 * 3.14159265358979323846) * s_range(&cs, 0.5, 2.0);
    for (int l = 0; l < 4; ++l) cpg[12 + l] = s_range(&cs, -0.5, 0.5);
    for (int l = 0; l < 4; ++l) cpg[l] = s_range(&cs, -0.1, 0.1);
    for (int l = 0; l < 4; ++l) cpg[4 + l] = 0.0;
    return 0;
}

/* One CPG step + physics step.  rest_base[12] holds the static rests and
 * L0 (indices 8..11); cpg = {x[4], y[4], omega[4], c[4]} updated in place. */
int hbo_cpg_step(double* pos, double* vel, const double* rest_base, double* cpg, double dt,
                 double* time) {
    if (!(dt > 0.0)) return -1;
    double nx[4];
    for (int l = 0; l < 4; ++l)
        nx[l] = cpg[l] + dt * (cpg[8 + l] * cpg[4 + l] + cpg[12 + l] * cpg[(l + 1) & 3]);
    for (int l = 0; l < 4; ++l) {
        cpg[4 + l] = cpg[4 + l] - dt * (cpg[8 + l] * nx[l]);
        cpg[l] = nx[l];
    }
    double rest[12];
    for (int k = 0; k < 8; ++k) rest[k] = rest_base[k];
    for (int l = 0; l < 4; ++l) {
        const double x = cpg[l];
        const double u = (x < -1.0) ? -1.0 : ((x > 1.0) ? 1.0 : x);
        rest[8 + l] = rest_base[8 + l] * (1.0 + 0.2 * u);
    }
    return hbo_step(HBO_CPG_HINGE, pos, vel, rest, dt, time);
}

int hbo_cpg_simulate(uint64_t seed, uint64_t steps, hbo_result* out, uint64_t* fail_step) {
    if (steps < 1) return -1;
    double pos[27], vel[27], rest[12], cpg[16];
    hbo_cpg_build(seed, pos, vel, rest, cpg);
    const double sx = pos[0], sy = pos[1];
    double time = 0.0;
    for (uint64_t s = 0; s < steps; ++s) {
        if (hbo_cpg_step(pos, vel, rest, cpg, 0.002, &time) == 1) {
            if (fail_step) *fail_step = s + 1;
            return 1;
        }
    }
    const double dx = pos[0] - sx, dy = pos[1] - sy;
    uint64_t h = hbo_checksum(9, pos, vel);
    for (int l = 0; l < 8; ++l) h = fnv_absorb(h, cpg[l]);
    out->seed = seed;
    out->fitness = sqrt(dx * dx + dy * dy);
    out->checksum = h;
    out->steps_executed = steps;
    if (fail_step) *fail_step = 0;
    return 0;
}
