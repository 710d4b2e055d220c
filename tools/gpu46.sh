timeout 900 python tools/streams_probe.py 20 > gpurun_out/streams_probe_r2v46.log 2>&1
