timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v72.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v72.log
timeout 1500 python bench.py --no-configs --no-slab --no-pipeline-pass > gpurun_out/bench_r2v72.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v72.log
