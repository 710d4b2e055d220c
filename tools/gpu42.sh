set -x
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v42.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v42.log
timeout 600 python tools/graph_probe.py > gpurun_out/graph_probe_r2v42.log 2>&1
KFBI_OP_CTA=0 timeout 600 python tools/graph_probe.py > gpurun_out/graph_probe_r2v42_grid.log 2>&1
