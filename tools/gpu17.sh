timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v18.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v18.log
timeout 1200 python bench.py --no-slab --no-configs > gpurun_out/bench_r2v18.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v18.log
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:"stencil_eval" -c 3 \
  -o gpurun_out/prof_seval3 -f python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline \
  --no-pipeline-pass --no-configs --no-slab --profile > gpurun_out/ncu_seval2.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_seval3.json gpurun_out/prof_seval3.ncu-rep > /dev/null 2>&1
rm -f gpurun_out/prof_seval3.ncu-rep
