# ncu: launch list of the timed region + full captures of the box passes in the bench
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
  --log-file gpurun_out/launches_r2v14.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline \
  --no-pipeline-pass --no-configs --no-slab --profile > gpurun_out/ncu_launch_r2v14.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"rows_fwd_reg|rows_inv_reg|cols_tri" -c 12 -o gpurun_out/prof_box_r2v14 -f \
  python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline --no-pipeline-pass --no-configs \
  --no-slab --profile > gpurun_out/ncu_full_r2v14.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_box_r2v14.json gpurun_out/prof_box_r2v14.ncu-rep > /dev/null 2>&1
python tools/traffic_json.py gpurun_out/ncu_traffic_r2v14.json gpurun_out/prof_box_r2v14.json > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"circ_block|spec_block|edges_spectral|corr_edges|op_solve|extract_update|heat_rhs|wave_rhs|nonlinear|mask_norm" -c 20 \
  -o gpurun_out/prof_rest_r2v14 -f python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline \
  --no-pipeline-pass --no-configs --no-slab --profile > gpurun_out/ncu_full2_r2v14.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_rest_r2v14.json gpurun_out/prof_rest_r2v14.ncu-rep > /dev/null 2>&1
if [ $(du -sm gpurun_out | cut -f1) -gt 56 ]; then rm -f gpurun_out/prof_rest_r2v14.ncu-rep; fi
