timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v25.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v25.log
timeout 1200 python bench.py --no-slab --no-configs > gpurun_out/bench_r2v25.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v25.log
bash tools/gpu20.sh
