#!/bin/bash
# Round profiling pass (run under gpurun; results in gpurun_out/, copy the
# ones to keep into profiles/):
#   bench_box.json          default bench line (configs[1]) incl. CPU baseline
#   bench_box_ref.json      the reference arm (bench.py --impl reference)
#   models_8192x5000.jsonl  every multi-body model at the configs[2] size
#   launches_box.csv        ncu launch list of the default bench command
#   prof_box.ncu-rep        ncu --set full capture of one box_kernel launch
#   bench_ea_*.json         configs[4] generation loop (box, box_and_ball) + reference arms
#   launches_ea_box.csv     ncu launch list of one box generation loop (sort / select / eval kernels)
#   sweeps.json             variant / step sweeps (tools/sweep.py)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_box.json 2> gpurun_out/bench_box.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_box_ref.json 2> gpurun_out/bench_box_ref.err
: > gpurun_out/models_8192x5000.jsonl
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  timeout 900 python bench.py --model $m --variants 8192 --sim-steps 5000 --steps 3 --warmup 3 \
    >> gpurun_out/models_8192x5000.jsonl 2> gpurun_out/models_$m.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_box.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:box_kernel -s 3 -c 1 \
  -o gpurun_out/prof_box -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full.log 2>&1
for m in box box_and_ball; do
  timeout 600 python bench.py --workload ea --model $m > gpurun_out/bench_ea_$m.json 2> /dev/null
  timeout 600 python bench.py --workload ea --model $m --impl reference > gpurun_out/bench_ea_${m}_ref.json 2> /dev/null
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_ea_box.csv python bench.py --workload ea --model box --steps 1 --warmup 3 \
  > /dev/null 2>&1
timeout 1800 python tools/sweep.py --out gpurun_out/sweeps.json > gpurun_out/sweep.log 2>&1
ls -la gpurun_out
