timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -k "headline or full_runs or interface or pipeline_solve" tests/test_gpu_graph.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v103.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v103.log
for c in 1 0; do
KFBI_SPEC_CLUSTER=$c timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spec_block" -c 8 --csv --log-file gpurun_out/speccl${c}_r2v103.csv python bench.py --no-configs --no-slab --no-pipeline-pass --steps 1 --warmup 3 --sequential > /dev/null 2>&1
done
timeout 900 python bench.py --no-configs --no-pipeline-pass > gpurun_out/bench_r2v103.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v103.log
