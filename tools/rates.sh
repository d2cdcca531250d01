timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread > gpurun_out/pytest_gpu_p.log 2>&1; tail -n 2 gpurun_out/pytest_gpu_p.log
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  for v in 8192 32768 131072; do
    timeout 600 python bench.py --model $m --variants $v --sim-steps 1000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null |
      python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$m $v %.4e vs/s frac %.3f replays %d %s' % (d['value'], r['frac'], r['exact_step_replays'], r['kernel']))"
  done
done
