mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench.py -q --timeout 600 > gpurun_out/pytest_bench.log 2>&1
tail -n 3 gpurun_out/pytest_bench.log
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  timeout 600 python bench.py --model $m --variants 32768 --sim-steps 1000 --steps 3 --warmup 3 --no-cpu-baseline --precision fp32 2>/dev/null
done > gpurun_out/bench_fp32_32768.jsonl
python -c "
import json
for l in open('gpurun_out/bench_fp32_32768.jsonl'):
    d=json.loads(l); print(d['config']['model'], '%.4g'%d['value'], d['roofline']['frac'], d['fp32'])"
