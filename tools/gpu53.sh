timeout 900 python tools/streams_probe.py 20 > gpurun_out/streams_probe_r2v53.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v53.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v53.log
