# round-2 GPU pass: full GPU test suite (per-test timeout), benches, tuning
timeout 1500 python -m pytest tests -m gpu -v --timeout 300 --timeout-method thread --durations 30 > gpurun_out/pytest_gpu.log 2>&1
grep -E "passed|failed|FAILED|ERROR|Timeout" gpurun_out/pytest_gpu.log | tail -15
timeout 300 python bench.py > gpurun_out/bench_box.json 2> gpurun_out/bench_box.err
timeout 600 python bench.py --model cpg_hinge --variants 8192 --sim-steps 5000 --steps 3 --warmup 3 > gpurun_out/bench_cpg.json 2> gpurun_out/bench_cpg.err
timeout 1200 bash tools/tune_minb.sh "arm_with_rope cpg_hinge box_and_ball" "32768 131072" 1000 > gpurun_out/tune_minb.txt 2>&1
cat gpurun_out/tune_minb.txt
