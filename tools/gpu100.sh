timeout 1500 ncu --set full --clock-control none --profile-from-start off -k regex:"rows_fwd_facr|cols_tri|rows_inv_reg|rows_odd_facr" -c 24 \
  -o /tmp/prof_traffic -f python bench.py --steps 1 --warmup 3 --repeats 1 --no-configs --no-slab --no-pipeline-pass --profile --sequential > gpurun_out/prof_traffic_r2v100.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_traffic_r2v100.json /tmp/prof_traffic.ncu-rep > /dev/null 2>&1
