set -x
timeout 600 python tools/graph_debug.py > gpurun_out/graph_debug_r2v40.log 2>&1
timeout 600 python tools/graph_probe.py > gpurun_out/graph_probe_r2v40.log 2>&1
