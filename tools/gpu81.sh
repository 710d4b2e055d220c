timeout 900 python -m pytest tests/test_gpu_parity.py -k "facr_trace" tests/test_gpu_tri.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v81.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v81.log
timeout 900 python bench.py --no-configs --no-pipeline-pass --steps 5 --warmup 3 > gpurun_out/bench_r2v81.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v81.log
