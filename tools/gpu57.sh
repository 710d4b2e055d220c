timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rows_fwd_facr|rows_inv_reg|rows_odd" -c 3 \
  -o /tmp/prof_rows -f python tools/prof_jumps.py 4096 heat > gpurun_out/prof_rows_r2v57.log 2>&1
for kn in rows_fwd_facr rows_inv_reg rows_odd_facr; do
ncu -i /tmp/prof_rows.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:$kn --launch-count 1 > gpurun_out/src_${kn}_r2v57.csv 2>&1
done
ls -la gpurun_out/src_*_r2v57.csv >> gpurun_out/prof_rows_r2v57.log
