timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"op_solve_pair_kernel|op_solve_half" -s 3 -c 2 \
  -o /tmp/prof_op -f python bench.py --no-configs --no-slab --no-pipeline-pass --steps 1 --warmup 3 --sequential > gpurun_out/prof_op_r2v82.log 2>&1
ncu -i /tmp/prof_op.ncu-rep --page raw --csv > gpurun_out/raw_op_r2v82.csv 2>&1
ncu -i /tmp/prof_op.ncu-rep --page details --csv > gpurun_out/details_op_r2v82.csv 2>&1
ncu -i /tmp/prof_op.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:op_solve_pair --launch-count 1 > gpurun_out/src_op_pair_r2v82.csv 2>&1
cp /tmp/prof_op.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out/*r2v82* >> gpurun_out/prof_op_r2v82.log
