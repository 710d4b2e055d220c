set -x
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_headline.py -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_r2v32.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v32.log
timeout 600 python tools/check_box.py 256 1024 2048 4096 8192 16384 > gpurun_out/box_r2v32.log 2>&1
KFBI_EDGES_SMEM=0 timeout 600 python tools/edges_probe.py save > gpurun_out/edges_r2v32.log 2>&1
timeout 600 python tools/edges_probe.py >> gpurun_out/edges_r2v32.log 2>&1
