// hb_internal.h — interface between the host runtime (hb_runtime.cpp) and
// the kernels (hb_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/hbgpu.h"

namespace hb {

// One batch on one device.  init: SoA rows (state_rows(kind) x ld doubles),
// read-only.  out / fail: n entries.  final_state (nullable): SoA rows.
struct SimArgs {
    const double* init;
    size_t n;
    size_t ld;
    uint64_t steps;
    double dt;
    const uint64_t* seeds;  // device pointer, nullable
    hb_variant_result* out;
    uint64_t* fail;
    double* final_state;
};

cudaError_t launch_sim(int kind, const SimArgs& a, cudaStream_t st, int sms);
const char* kernel_name(int kind, size_t n);
cudaError_t launch_fp64_probe(double* scratch, int sms, int iters, cudaStream_t st, double* ops);

}  // namespace hb
