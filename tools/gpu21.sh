timeout 1200 python -m pytest tests/test_gpu_tri.py -q -x --tb=short -p no:cacheprovider -k "facr" > gpurun_out/pytest_facr4.log 2>&1; echo rc=$? >> gpurun_out/pytest_facr2.log
bash tools/gpu20.sh
timeout 1200 python bench.py --no-slab --no-configs > gpurun_out/bench_r2v23.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v21.log
