timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -m gpu -q --tb=short -p no:cacheprovider -k "full_runs or graph or runs_1024" > gpurun_out/pytest_r2v49.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v49.log
timeout 1500 python bench.py --no-configs --no-slab --no-pipeline-pass > gpurun_out/bench_r2v49.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v49.log
