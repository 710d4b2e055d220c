timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2v106.log 2>&1; echo rc=$? >> gpurun_out/smoke_r2v106.log
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v106.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v106.log
timeout 1200 python bench.py > gpurun_out/bench_r2v106.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v106.log
