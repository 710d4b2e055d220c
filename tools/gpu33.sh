set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spec_block|edges_spectral|circ_block|group_sums" -c 8 \
  -o gpurun_out/prof_jumps_heat -f python tools/prof_jumps.py 4096 heat > gpurun_out/prof_jumps_heat.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_jumps_heat.json gpurun_out/prof_jumps_heat.ncu-rep > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rows_odd|corr_edges" -c 4 \
  -o gpurun_out/prof_odd_schr -f python tools/prof_jumps.py 4096 schrodinger > gpurun_out/prof_odd_schr.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_odd_schr.json gpurun_out/prof_odd_schr.ncu-rep > /dev/null 2>&1
