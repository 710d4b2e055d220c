timeout 120 ./tools/mb/gsync2 > gpurun_out/gsync2_r2v56.log 2>&1
