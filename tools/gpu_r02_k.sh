# round-2 robustness pass: compute-sanitizer over every kernel family (incl.
# the two-lane CpgHinge and the register-capped shapes), smoke(), the
# multi-rank bench path (2 ranks over gloo on one GPU), the configs[3] step
# sweep through the reference harness with start-up reservation
mkdir -p gpurun_out/ref_sweep
{
echo "# compute-sanitizer over tools/sanitize_probe.py, B200, round 2"
for t in memcheck racecheck synccheck; do
  echo "## $t"
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_probe.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|Error|error|hazard" | head -20
done
} > gpurun_out/compute_sanitizer.txt 2>&1
cat gpurun_out/compute_sanitizer.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 2 gpurun_out/smoke.log
HB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
tail -c 600 gpurun_out/bench_2rank_gloo.json
HB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --workload ea --steps 3 --warmup 3 > gpurun_out/bench_ea_2rank_gloo.json 2> gpurun_out/bench_ea_2rank_gloo.err
tail -c 400 gpurun_out/bench_ea_2rank_gloo.json
timeout 1500 oracle/_ref/ref_sweep tools/sweeps/b200_step_sweep.toml gpurun_out/ref_sweep/step_sweep > gpurun_out/ref_sweep/step_sweep.log 2>&1
tail -n 3 gpurun_out/ref_sweep/step_sweep.log
