#!/bin/bash
# One-GPU profiling pass (run under gpurun): per-model kernel timings, the
# ncu launch list of the default bench command, and one --set full capture.
set -x
mkdir -p gpurun_out
for m in box box_and_ball arm_with_rope humanoid; do
  case $m in box) v=16384; s=1000;; box_and_ball) v=16384; s=1000;; arm_with_rope) v=8192; s=1000;; humanoid) v=8192; s=200;; esac
  timeout 300 python bench.py --model $m --variants $v --sim-steps $s --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$m.json 2>gpurun_out/bench_$m.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:box_kernel -s 3 -c 1 -o gpurun_out/prof_box python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:humanoid_pair -s 3 -c 1 -o gpurun_out/prof_humanoid python bench.py --model humanoid --variants 8192 --sim-steps 200 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_h.log 2>&1
ls -la gpurun_out
