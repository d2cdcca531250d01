#!/bin/bash
# Humanoid variants: prediction in registers vs shared memory (HB_HUMANOID_SQ), sweep groups.
for n in 8192 32768; do
  for sq in 0 1; do for u in 1 2; do
    r=$(HB_HUMANOID_SQ=$sq HB_UNROLL_HUMANOID=$u timeout 300 python bench.py --model humanoid --variants $n --sim-steps 200 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('%.4e vs/s %.3f ms frac %.3f replays %d' % (d['value'], d['ms_per_step'], r['frac'], r['exact_step_replays']))")
    echo "n=$n SQ=$sq U=$u $r"
  done; done
done
