#!/bin/bash
# ncu --set full capture of one model's stepping kernel (run under gpurun).
#   tools/ncu_model.sh <model> <variants> <sim_steps> <kernel-regex> <out-name>
m=$1; v=$2; s=$3; k=$4; o=$5
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
  -o gpurun_out/$o python bench.py --model $m --variants $v --sim-steps $s --steps 1 --warmup 2 \
  --no-cpu-baseline --no-e2e > gpurun_out/$o.log 2>&1
