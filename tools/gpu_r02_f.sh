# parity after the RANGED certificate + wave balancing; balance A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu_f.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_f.log
timeout 1200 bash tools/tune_balance.sh "box_and_ball" "32768 131072 262144" 1000 "0 12 16" > gpurun_out/tune_balance_bb.txt 2>&1
timeout 1500 bash tools/tune_balance.sh "arm_with_rope cpg_hinge humanoid" "32768 131072" 1000 > gpurun_out/tune_balance.txt 2>&1
cat gpurun_out/tune_balance_bb.txt gpurun_out/tune_balance.txt
