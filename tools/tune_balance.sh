#!/bin/bash
# Wave balancing (HB_BALANCE) x register cap (HB_MINB) A/B of the multi-body
# kernels (run under gpurun): kernel rate per (model, variants, MB, balance).
#   tools/tune_balance.sh "<models>" "<variant counts>" [sim_steps] [minb list]
models=${1:-"box_and_ball arm_with_rope cpg_hinge humanoid"}
sizes=${2:-"32768 131072"}
s=${3:-1000}
mbs=${4:-"0"}
for m in $models; do
  M=$(echo $m | tr a-z A-Z)
  for v in $sizes; do
    for mb in $mbs; do
      for bal in 0 1; do
        envs="HB_BALANCE=$bal"
        [ "$mb" != 0 ] && envs="$envs HB_MINB_$M=$mb"
        r=$(env $envs timeout 300 python bench.py --model $m --variants $v \
              --sim-steps $s --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null |
            python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('%.4e vs/s  %.3f ms  frac %.3f replays %d' % (d['value'], d['ms_per_step'], r['frac'], r['exact_step_replays']))")
        echo "$m n=$v MB=$mb balance=$bal $r"
      done
    done
  done
done
