timeout 900 ncu --set full --clock-control none --import-source on -k regex:"nonlinear_phase|mask_norm" -s 2 -c 3 \
  -o /tmp/prof_schr -f python tools/schr_steps.py 4 > gpurun_out/prof_schr_r2v69.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_schr_r2v69.json /tmp/prof_schr.ncu-rep > /dev/null 2>&1
ncu -i /tmp/prof_schr.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:nonlinear_phase --launch-count 1 > gpurun_out/src_nonlinear_r2v69.csv 2>&1
