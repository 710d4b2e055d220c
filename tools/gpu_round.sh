#!/bin/bash
# One gpurun session: smoke, GPU tests, bench, ncu launch list + one full capture.
# Usage (from the repo root, on the GPU box): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench_$TAG.log 2>&1; echo "rc=$?" >> $OUT/bench_$TAG.log
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --profile-from-start off --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile > $OUT/ncu_launch_bench_$TAG.log 2>&1
  echo "rc=$?" >> $OUT/ncu_launch_bench_$TAG.log
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:cols_ -c 4 \
    -o $OUT/prof_cols_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile --equations heat,schrodinger > $OUT/ncu_full_$TAG.log 2>&1
  echo "rc=$?" >> $OUT/ncu_full_$TAG.log
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"rows_fwd|rows_inv|corr_edges|op_solve|heat_rhs|nonlinear|schr_ustar|wave_rhs|jumps" -c 14 \
    -o $OUT/prof_rows_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile > $OUT/ncu_full2_$TAG.log 2>&1
  echo "rc=$?" >> $OUT/ncu_full2_$TAG.log
fi
# summaries on the box; keep the merged-back directory under gpurun's 64 MiB cap
for r in $OUT/prof_cols_$TAG.ncu-rep $OUT/prof_rows_$TAG.ncu-rep; do
  [ -f $r ] && python tools/ncu_summary.py ${r%.ncu-rep}.json $r > /dev/null 2>&1
done
python tools/traffic_json.py $OUT/prof_cols_$TAG.json $OUT/ncu_traffic_$TAG.json > /dev/null 2>&1
if [ $(du -sm $OUT | cut -f1) -gt 56 ]; then rm -f $OUT/prof_rows_$TAG.ncu-rep; fi
if [ $(du -sm $OUT | cut -f1) -gt 56 ]; then rm -f $OUT/prof_cols_$TAG.ncu-rep; fi
