timeout 900 python tools/c3_probe.py > gpurun_out/c3_probe_r2v63.log 2>&1
