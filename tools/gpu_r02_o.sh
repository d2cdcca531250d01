# arm in the latency regime (8 192 / 32 768): ncu stall profile, and the
# sweep-unroll factor at those sizes
mkdir -p gpurun_out/ncu
bash tools/ncu_model.sh arm_with_rope 8192 500 multibody prof_arm8k
bash tools/ncu_model.sh arm_with_rope 32768 200 multibody prof_arm32k
for f in gpurun_out/prof_arm8k.ncu-rep gpurun_out/prof_arm32k.ncu-rep; do
  b=$(basename $f .ncu-rep); python tools/ncu_summary.py $f > gpurun_out/ncu/$b.summary.txt 2>&1
  ncu -i $f --page source --csv > gpurun_out/ncu/$b.source.csv 2>/dev/null; gzip -f gpurun_out/ncu/$b.source.csv; rm -f $f
done
cat gpurun_out/ncu/prof_arm8k.summary.txt gpurun_out/ncu/prof_arm32k.summary.txt | grep -E "duration|issue_active|fp64_cycles_active.avg.pct_of_peak_sustained_active|warps_active|registers|stalls|inst_executed.sum"
for v in 8192 32768; do for u in 1 2 4 8; do
  HB_UNROLL_ARM_WITH_ROPE=$u timeout 300 python bench.py --model arm_with_rope --variants $v --sim-steps 1000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null |
    python -c "import json,sys; d=json.load(sys.stdin); print('arm $v U=$u %.4e' % d['value'])"
done; done
