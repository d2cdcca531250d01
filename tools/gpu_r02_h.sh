# round-2 measurement pass on the final kernels: GPU tests, the round
# profile (benches, models, EA, launch lists, sweeps), the reference harness
# sweeps with start-up reservation, FP32 mode.
mkdir -p gpurun_out/ref_sweep
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread --durations 15 > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_ea.py -q -s -k eight_contexts > gpurun_out/ea8_overhead.log 2>&1
grep "8 contexts" gpurun_out/ea8_overhead.log
timeout 2700 bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 300 python tools/fp32_mode.py > gpurun_out/fp32_mode.json 2> gpurun_out/fp32_mode.err
timeout 2400 oracle/_ref/ref_sweep tools/sweeps/b200_variant_grid.toml gpurun_out/ref_sweep/variant_grid > gpurun_out/ref_sweep/variant_grid.log 2>&1
tail -n 4 gpurun_out/ref_sweep/variant_grid.log
du -sh gpurun_out
