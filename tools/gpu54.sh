timeout 900 python tools/host_profile.py 20 > gpurun_out/host_profile_r2v54.log 2>&1
