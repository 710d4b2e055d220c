set -x
for eq in heat schrodinger; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spec_block|edges_spectral|circ_block|group_sums|corr_edges" -c 12 --csv \
  --log-file gpurun_out/jumps_times_${eq}_r2v35.csv python tools/prof_jumps.py 4096 $eq > /dev/null 2>&1
done
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_r2v35.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v35.log
timeout 1500 python bench.py --no-configs --no-slab > gpurun_out/bench_r2v35.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v35.log
