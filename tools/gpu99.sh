timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rows_|cols_|op_solve" -s 20 -c 12 \
  -o /tmp/prof_bench -f python bench.py --steps 2 --warmup 3 --repeats 1 --no-configs --no-slab --no-pipeline-pass --sequential > gpurun_out/prof_bench_r2v99.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_bench_r2v99.json /tmp/prof_bench.ncu-rep > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2v99.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-configs --no-slab --no-pipeline-pass --profile --sequential > gpurun_out/launches_r2v99.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_streams_r2v99.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-configs --no-slab --no-pipeline-pass --profile > gpurun_out/launches_streams_r2v99.log 2>&1
