# ncu captures, tuning at the knee, the paper's sweeps through the reference harness
bash tools/prof_r02.sh > gpurun_out/prof.log 2>&1
timeout 900 bash tools/tune_minb.sh "arm_with_rope cpg_hinge" "65536 262144" 1000 > gpurun_out/tune_minb2.txt 2>&1
mkdir -p gpurun_out/ref_sweep
timeout 1500 oracle/_ref/ref_sweep tools/sweeps/b200_step_sweep.toml gpurun_out/ref_sweep/step_sweep > gpurun_out/ref_sweep/step_sweep.log 2>&1
timeout 2400 oracle/_ref/ref_sweep tools/sweeps/b200_variant_grid.toml gpurun_out/ref_sweep/variant_grid > gpurun_out/ref_sweep/variant_grid.log 2>&1
cat gpurun_out/tune_minb2.txt; tail -5 gpurun_out/ref_sweep/*.log; ls gpurun_out/ref_sweep/*
