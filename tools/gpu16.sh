timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:"stencil_eval" -c 3 \
  -o gpurun_out/prof_seval -f python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline \
  --no-pipeline-pass --no-configs --no-slab --profile > gpurun_out/ncu_seval.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_seval.json gpurun_out/prof_seval.ncu-rep > /dev/null 2>&1
python tools/ncu_src.py gpurun_out/prof_seval.ncu-rep stencil_eval 30 > gpurun_out/seval_src.txt 2>&1
