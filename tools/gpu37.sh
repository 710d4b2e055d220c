set -x
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_slab.py tests/test_gpu_stepping.py -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_r2v37.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v37.log
for i in 1 2 3; do
timeout 1500 python bench.py --no-configs --no-slab --no-pipeline-pass > gpurun_out/bench_r2v37_$i.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v37_$i.log
done
