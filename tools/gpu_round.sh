# round measurement pass (run under gpurun from the repo root): GPU tests, sanitizer,
# the round profile, saturated rates, FP32-mode lines, ncu captures
# (summarised on the box; .ncu-rep files are too large to ship back)
mkdir -p gpurun_out/ncu
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread --durations 10 > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
{
echo "# compute-sanitizer over tools/sanitize_probe.py (every model incl. the two-lane CpgHinge and humanoid, the register-capped 65 536-variant shapes, run_ea queued / device sort / BoxAndBall, FP32 mode, generic variant, Box zero-copy, hb_ctx_reserve), B200, round 2"
for t in memcheck racecheck synccheck; do
  echo "## $t"
  timeout 1200 compute-sanitizer --tool $t --print-limit 5 python tools/sanitize_probe.py 2>&1 | grep -E "SUMMARY|Race reported|Error:" | head -12
done
} > gpurun_out/compute_sanitizer.txt 2>&1
cat gpurun_out/compute_sanitizer.txt
timeout 2700 bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
timeout 600 python bench.py --model cpg_hinge --variants 8192 --sim-steps 5000 --steps 3 --warmup 3 > gpurun_out/bench_cpg.json 2> gpurun_out/bench_cpg.err
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  for v in 131072 262144; do
    timeout 600 python bench.py --model $m --variants $v --sim-steps 1000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null |
      python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$m $v %.4e vs/s frac %.3f replays %d %s' % (d['value'], r['frac'], r['exact_step_replays'], r['kernel']))"
  done
done > gpurun_out/saturated.txt
for m in box_and_ball arm_with_rope humanoid cpg_hinge; do
  timeout 600 python bench.py --model $m --variants 32768 --sim-steps 1000 --steps 3 --warmup 3 --no-cpu-baseline --precision fp32 2>/dev/null
done > gpurun_out/bench_fp32_32768.jsonl
bash tools/prof_r02.sh > gpurun_out/prof.log 2>&1
for f in gpurun_out/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python tools/ncu_summary.py $f > gpurun_out/ncu/$b.summary.txt 2>&1
  rm -f $f
done
cat gpurun_out/saturated.txt
du -sh gpurun_out
# the paper's sweeps through the reference's own harness (tools/ref_sweep.cpp)
mkdir -p gpurun_out/ref_sweep
timeout 1500 oracle/_ref/ref_sweep tools/sweeps/b200_step_sweep.toml gpurun_out/ref_sweep/step_sweep > gpurun_out/ref_sweep/step_sweep.log 2>&1
timeout 2400 oracle/_ref/ref_sweep tools/sweeps/b200_variant_grid.toml gpurun_out/ref_sweep/variant_grid > gpurun_out/ref_sweep/variant_grid.log 2>&1
for f in gpurun_out/ref_sweep/*.log; do tail -n 2 $f; done
