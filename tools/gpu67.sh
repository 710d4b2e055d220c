KFBI_EDGES_FULL=0 timeout 600 python tools/edges_probe.py save > gpurun_out/edges_r2v67.log 2>&1
timeout 600 python tools/edges_probe.py >> gpurun_out/edges_r2v67.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_headline.py -m gpu -q --tb=short -p no:cacheprovider -k "staged or schrodinger" > gpurun_out/pytest_r2v67.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v67.log
