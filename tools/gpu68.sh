timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2v68.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-configs --no-slab --no-pipeline-pass --profile --sequential > gpurun_out/launches_r2v68.log 2>&1
