#!/bin/bash
# Kernel (and e2e) rates of every model at the config-3 size, one line each.
# usage: tools/models_bench.sh [variants] [sim_steps]
v=${1:-8192}; s=${2:-500}
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  timeout 300 python bench.py --model $m --variants $v --sim-steps $s --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', $v, $s, '%.4g' % d['value'], 'frac %.4f' % d['roofline']['frac'], 'e2e %.4g' % d['e2e']['value'], 'replays', d['roofline']['exact_step_replays'])"
done
