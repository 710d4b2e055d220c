timeout 1200 python -m pytest tests/test_gpu_tri.py tests/test_gpu_headline.py tests/test_gpu_parity.py -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v24.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v24.log
timeout 1200 python bench.py --no-slab --no-configs > gpurun_out/bench_r2v24.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v24.log
