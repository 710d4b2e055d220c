set -x
for eq in heat schrodinger; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rows_|cols_" -c 8 \
  -o gpurun_out/prof_facr_$eq -f python tools/prof_jumps.py 4096 $eq > gpurun_out/prof_facr_${eq}.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_facr_$eq.json gpurun_out/prof_facr_$eq.ncu-rep > /dev/null 2>&1
python tools/ncu_src.py gpurun_out/prof_facr_$eq.ncu-rep "rows_fwd_facr" 20 > gpurun_out/prof_facr_${eq}_src.txt 2>&1
rm -f gpurun_out/prof_facr_$eq.ncu-rep
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2v48.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-configs --no-slab --no-pipeline-pass --profile > gpurun_out/launches_r2v48.log 2>&1
