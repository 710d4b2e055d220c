timeout 900 python tools/e2e_probe.py 20 > gpurun_out/e2e_probe_r2v45.log 2>&1
