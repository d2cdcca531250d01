/* hb_oracle.h — TEST INFRASTRUCTURE ONLY (see hb_oracle.c header). */
#ifndef HB_ORACLE_H
#define HB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { HBO_BOX = 0, HBO_BOX_AND_BALL = 1, HBO_ARM_WITH_ROPE = 2, HBO_HUMANOID = 3, HBO_CPG_HINGE = 4 };

/* Layout-identical to hetbench::VariantResult (simkernel.hpp:51-58). */
typedef struct {
    uint64_t seed;
    double fitness;
    uint64_t checksum;
    uint64_t steps_executed;
} hbo_result;

/* Field order of hetbench::AllocationPlan (scheduler.hpp:24-30). */
typedef struct {
    uint64_t n_total, n_cpu, n_accel;
    double accel_fraction, requested_accel_fraction;
} hbo_plan;

uint64_t hbo_mix64(uint64_t x);
uint64_t hbo_rng_at(uint64_t key, uint64_t counter);
double hbo_to_unit(uint64_t bits);
int hbo_body_count(int kind);
int hbo_constraint_count(int kind);
int hbo_topology(int kind, int* ca, int* cb, double* stiff);
int hbo_build_model(int kind, uint64_t seed, double* pos, double* vel, double* rest);
int hbo_step(int kind, double* pos, double* vel, const double* rest, double dt, double* time);
uint64_t hbo_checksum(int n, const double* pos, const double* vel);
int hbo_simulate(int kind, uint64_t seed, uint64_t steps, hbo_result* out, uint64_t* fail_step);
double hbo_time_after(uint64_t steps, double dt);
int hbo_blowup_message(uint64_t seed, uint64_t fail_step, double dt, char* buf, size_t cap);
int hbo_simulate_batch(int kind, const uint64_t* seeds, size_t n, uint64_t steps, int threads,
                       hbo_result* out, uint64_t* fail_step);
int hbo_plan_allocation(double t_cpu, double t_accel, int cpu_ok, int accel_ok, uint64_t n_total,
                        hbo_plan* plan);
void hbo_stable_order_desc(const double* fitness, size_t n, size_t* order);
uint64_t hbo_init_genome(uint64_t seed, uint64_t i);
uint64_t hbo_child_genome(uint64_t parent, uint64_t g, uint64_t i);
/* CPG / hinge model (kind 4, not in the reference; see hb_oracle.c). */
int hbo_cpg_build(uint64_t seed, double* pos, double* vel, double* rest, double* cpg);
int hbo_cpg_step(double* pos, double* vel, const double* rest_base, double* cpg, double dt,
                 double* time);
int hbo_cpg_simulate(uint64_t seed, uint64_t steps, hbo_result* out, uint64_t* fail_step);
int hbo_run_ea(int kind, size_t pop, uint64_t generations, uint64_t steps, uint64_t seed,
               int threads, uint64_t* genomes, double* fitness);

#ifdef __cplusplus
}
#endif
#endif
