# round-2 GPU pass after a container rebuild: headline benches, round-2 ncu
# captures (summarised on the box; the .ncu-rep files are too large to ship
# back), the paper's sweeps through the reference harness.
mkdir -p gpurun_out/ref_sweep gpurun_out/ncu
timeout 300 python bench.py > gpurun_out/bench_box.json 2> gpurun_out/bench_box.err
timeout 600 python bench.py --model cpg_hinge --variants 8192 --sim-steps 5000 --steps 3 --warmup 3 > gpurun_out/bench_cpg.json 2> gpurun_out/bench_cpg.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_box_reference.json 2> gpurun_out/bench_box_reference.err
bash tools/prof_r02.sh > gpurun_out/prof.log 2>&1
for f in gpurun_out/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python tools/ncu_summary.py $f > gpurun_out/ncu/$b.summary.txt 2>&1
  ncu -i $f --page raw --csv > gpurun_out/ncu/$b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv > gpurun_out/ncu/$b.source.csv 2>/dev/null
  gzip -f gpurun_out/ncu/$b.source.csv
  rm -f $f
done
timeout 1500 oracle/_ref/ref_sweep tools/sweeps/b200_step_sweep.toml gpurun_out/ref_sweep/step_sweep > gpurun_out/ref_sweep/step_sweep.log 2>&1
timeout 2400 oracle/_ref/ref_sweep tools/sweeps/b200_variant_grid.toml gpurun_out/ref_sweep/variant_grid > gpurun_out/ref_sweep/variant_grid.log 2>&1
for f in gpurun_out/ref_sweep/*.log; do tail -n 3 $f; done
du -sh gpurun_out; du -a gpurun_out | sort -n | tail -8
