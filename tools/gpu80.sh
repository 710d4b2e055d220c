timeout 900 python -m pytest tests/test_gpu_parity.py -k "facr_trace" -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v80a.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v80a.log
timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_tri.py tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v80.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v80.log
timeout 1500 python bench.py > gpurun_out/bench_r2v80.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v80.log
