#!/bin/bash
# Round-2 profiling pass for the multi-body kernels (run under gpurun):
# ncu --set full of one launch each — cpg_hinge at the configs[2] size
# (two-lane latency kernel), box_and_ball / arm_with_rope / cpg_hinge at
# 131 072 (throughput regime) — plus the launch list of the default bench.
mkdir -p gpurun_out
cap() {  # model variants steps out [env...]
  m=$1; v=$2; s=$3; o=$4; shift 4
  env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"multibody|cpg_pair" \
    -s 2 -c 1 -o gpurun_out/$o -f python bench.py --model $m --variants $v --sim-steps $s --steps 1 \
    --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/$o.log 2>&1
}
cap cpg_hinge 8192 1000 prof_cpg_pair
cap box_and_ball 131072 200 prof_bb131k
cap arm_with_rope 131072 100 prof_arm131k
cap cpg_hinge 131072 100 prof_cpg131k
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_box.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:box_kernel -s 3 -c 1 \
  -o gpurun_out/prof_box -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
