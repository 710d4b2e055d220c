timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_gmres.py -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v15.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v15.log
timeout 1200 python bench.py --no-slab > gpurun_out/bench_r2v15.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v15.log
timeout 900 ncu --set full --clock-control none --profile-from-start off \
  -k regex:"rows_fwd_reg<1|rows_inv_reg<1|cols_tri<1" -c 3 -o gpurun_out/prof_c128_r2v15 -f \
  python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline --no-pipeline-pass --no-configs \
  --no-slab --profile --equations schrodinger > gpurun_out/ncu_c128_r2v15.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_c128_r2v15.json gpurun_out/prof_c128_r2v15.ncu-rep > /dev/null 2>&1
python tools/traffic_json.py gpurun_out/ncu_traffic_r2v15.json profiles/r2_v14_ncu_box_passes.json gpurun_out/prof_c128_r2v15.json > /dev/null 2>&1
rm -f gpurun_out/prof_c128_r2v15.ncu-rep
