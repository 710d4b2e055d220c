set -x
KFBI_EDGES_SMEM=0 timeout 600 python tools/edges_probe.py save > gpurun_out/edges_r2v31.log 2>&1
timeout 600 python tools/edges_probe.py >> gpurun_out/edges_r2v31.log 2>&1
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_r2v31.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v31.log
timeout 1500 python bench.py > gpurun_out/bench_r2v31.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v31.log
