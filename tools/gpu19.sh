timeout 1200 python -m pytest tests/test_gpu_tri.py -q -x --tb=short -p no:cacheprovider -k "facr" > gpurun_out/pytest_facr.log 2>&1; echo rc=$? >> gpurun_out/pytest_facr.log
timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v19.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v19.log
KFBI_COLS=tridiagonal timeout 600 python tools/check_box.py 1024 2048 4096 8192 > gpurun_out/check_box_facr.log 2>&1
timeout 1200 python bench.py --no-slab --no-configs > gpurun_out/bench_r2v19.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v19.log
