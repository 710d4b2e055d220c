timeout 300 python tools/c2_probe.py > gpurun_out/c2_probe_r2v90.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v90.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v90.log
for sp in 1 0; do
KFBI_EDGE_SPLIT=$sp timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"edges_spectral_res" -c 8 --csv --log-file gpurun_out/esplit${sp}_r2v90.csv python bench.py --no-configs --no-slab --no-pipeline-pass --steps 1 --warmup 3 --sequential > /dev/null 2>&1
done
timeout 900 python bench.py --no-slab --no-pipeline-pass > gpurun_out/bench_r2v90.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v90.log
