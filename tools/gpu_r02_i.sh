# after moving the ranged-certificate precondition to a predicate
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu_i.log 2>&1
tail -n 2 gpurun_out/pytest_gpu_i.log
: > gpurun_out/models_8192x5000_i.jsonl
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  timeout 900 python bench.py --model $m --variants 8192 --sim-steps 5000 --steps 3 --warmup 3 \
    >> gpurun_out/models_8192x5000_i.jsonl 2> /dev/null
done
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  for v in 32768 131072; do
    timeout 600 python bench.py --model $m --variants $v --sim-steps 1000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null |
      python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$m $v %.4e vs/s frac %.3f replays %d' % (d['value'], r['frac'], r['exact_step_replays']))"
  done
done > gpurun_out/saturated_i.txt
cat gpurun_out/saturated_i.txt
python -c "
import json
for l in open('gpurun_out/models_8192x5000_i.jsonl'):
    d=json.loads(l); print(d['config']['model'], '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'])"
