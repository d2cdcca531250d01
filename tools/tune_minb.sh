#!/bin/bash
# Register-cap x sweep-unroll tuning of the multi-body kernels (run under
# gpurun): kernel rate per (model, variants, U, MB), one line each.
#   tools/tune_minb.sh "<models>" "<variant counts>" [sim_steps]
models=${1:-"box_and_ball arm_with_rope cpg_hinge"}
sizes=${2:-"32768 131072"}
s=${3:-1000}
for m in $models; do
  M=$(echo $m | tr a-z A-Z)
  case $m in cpg_hinge) us="1 2 4";; *) us="1 2 4 8";; esac
  for v in $sizes; do
    for u in $us; do
      for mb in 1 6 8; do
        if [ $mb != 1 ] && [ $u -gt 2 ]; then continue; fi
        r=$(env HB_UNROLL_$M=$u HB_MINB_$M=$mb timeout 300 python bench.py --model $m --variants $v \
              --sim-steps $s --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null |
            python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('%.4e vs/s  %.3f ms  frac %.3f replays %d' % (d['value'], d['ms_per_step'], r['frac'], r['exact_step_replays']))")
        echo "$m n=$v U=$u MB=$mb $r"
      done
    done
  done
done
