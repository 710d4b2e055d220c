timeout 600 python tools/graph_neumann_debug.py > gpurun_out/graph_neumann_r2v55.log 2>&1
