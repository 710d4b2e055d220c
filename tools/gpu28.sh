timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_headline.py -q -x --tb=short -p no:cacheprovider -k "facr or headline" > gpurun_out/pytest_r2v28.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v28.log
bash tools/gpu20.sh
timeout 1200 python bench.py --no-slab --no-configs > gpurun_out/bench_r2v28.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v28.log
