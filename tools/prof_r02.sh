#!/bin/bash
# Round-2 profiling pass for the multi-body kernels (run under gpurun):
# ncu --set full of one launch each — cpg_hinge at the configs[2] size
# (latency-bound), box_and_ball / arm_with_rope at 131 072 (throughput).
mkdir -p gpurun_out
cap() {  # model variants steps out [env...]
  m=$1; v=$2; s=$3; o=$4; shift 4
  env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:multibody -s 2 -c 1 \
    -o gpurun_out/$o -f python bench.py --model $m --variants $v --sim-steps $s --steps 1 --warmup 2 \
    --no-cpu-baseline --no-e2e > gpurun_out/$o.log 2>&1
}
cap cpg_hinge 8192 1000 prof_cpg
cap box_and_ball 131072 200 prof_bb131k
cap arm_with_rope 131072 100 prof_arm131k
cap arm_with_rope 131072 100 prof_arm131k_u1mb6 HB_UNROLL_ARM_WITH_ROPE=1 HB_MINB_ARM_WITH_ROPE=6
ls -la gpurun_out
