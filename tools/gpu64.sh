timeout 900 python tools/c3_profile.py > gpurun_out/c3_profile_r2v64.log 2>&1
