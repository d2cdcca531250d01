# humanoid one-warp CTAs + pair-shared rung rest lengths; cpg_pair replay sync
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread > gpurun_out/pytest_gpu_m.log 2>&1
tail -n 2 gpurun_out/pytest_gpu_m.log
{
echo "# compute-sanitizer over tools/sanitize_probe.py (every model incl. the two-lane CpgHinge and humanoid, the register-capped 65 536-variant shapes, run_ea queued / device sort / BoxAndBall, FP32 mode, generic variant, Box zero-copy, hb_ctx_reserve), B200, round 2"
for t in memcheck racecheck synccheck; do
  echo "## $t"
  timeout 1200 compute-sanitizer --tool $t --print-limit 5 python tools/sanitize_probe.py 2>&1 | grep -E "SUMMARY|Race reported|Error:" | head -12
done
} > gpurun_out/compute_sanitizer.txt 2>&1
cat gpurun_out/compute_sanitizer.txt
for m in humanoid cpg_hinge; do
  for v in 8192 32768 131072; do
    timeout 600 python bench.py --model $m --variants $v --sim-steps 1000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null |
      python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$m $v %.4e vs/s frac %.3f replays %d %s' % (d['value'], r['frac'], r['exact_step_replays'], r['kernel']))"
  done
done > gpurun_out/rates_m.txt
cat gpurun_out/rates_m.txt
