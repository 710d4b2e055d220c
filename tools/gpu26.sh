for eq in heat schrodinger; do
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"rows_fwd_facr|rows_inv_reg|cols_tri|rows_odd_facr" -c 8 -o gpurun_out/prof_facr_$eq -f \
  python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline --no-pipeline-pass --no-configs \
  --no-slab --profile --equations $eq > gpurun_out/ncu_facr_$eq.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_facr_$eq.json gpurun_out/prof_facr_$eq.ncu-rep > /dev/null 2>&1
done
python tools/traffic_json.py gpurun_out/ncu_traffic_r2v26.json gpurun_out/prof_facr_heat.json gpurun_out/prof_facr_schrodinger.json > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
  --log-file gpurun_out/launches_r2v26.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline \
  --no-pipeline-pass --no-configs --no-slab --profile > gpurun_out/ncu_launch_r2v26.log 2>&1
rm -f gpurun_out/prof_facr_schrodinger.ncu-rep
timeout 1200 python bench.py > gpurun_out/bench_r2v26.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v26.log
