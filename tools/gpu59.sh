timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_slab.py -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_r2v59.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v59.log
timeout 600 python tools/check_box.py 1024 2048 4096 8192 16384 > gpurun_out/box_r2v59.log 2>&1
