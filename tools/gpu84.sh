timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"spec_block|edges_spectral_res|circ_block" -s 12 -c 6 \
  -o /tmp/prof_spec -f python bench.py --no-configs --no-slab --no-pipeline-pass --steps 1 --warmup 3 --sequential > gpurun_out/prof_spec_r2v84.log 2>&1
ncu -i /tmp/prof_spec.ncu-rep --page details --csv > gpurun_out/details_spec_r2v84.csv 2>&1
ncu -i /tmp/prof_spec.ncu-rep --page raw --csv > gpurun_out/raw_spec_r2v84.csv 2>&1
for kn in spec_block edges_spectral_res circ_block; do
ncu -i /tmp/prof_spec.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:$kn --launch-count 1 > gpurun_out/src_${kn}_r2v84.csv 2>&1
done
