#!/bin/bash
# Sweep-unroll tuning (run under gpurun): kernel time per model per unroll factor.
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  case $m in box_and_ball) v=16384; s=1000; E=HB_UNROLL_BOX_AND_BALL;; arm_with_rope) v=8192; s=1000; E=HB_UNROLL_ARM_WITH_ROPE;; humanoid) v=8192; s=200; E=HB_UNROLL_HUMANOID;; cpg_hinge) v=8192; s=1000; E=HB_UNROLL_CPG_HINGE;; esac
  for u in 1 2 4 8; do  # (cpg_hinge: 1 2 4)
    r=$(env $E=$u timeout 300 python bench.py --model $m --variants $v --sim-steps $s --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('%.4e vs/s  %.3f ms  frac %.3f replays %d' % (d['value'], d['ms_per_step'], r['frac'], r['exact_step_replays']))")
    echo "$m U=$u $r"
  done
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('box %.4e vs/s  %.4f ms  frac %.3f' % (d['value'], d['ms_per_step'], r['frac']))"
