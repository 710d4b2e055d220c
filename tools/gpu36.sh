set -x
timeout 600 python -m pytest tests/test_slab.py -m gpu -q --tb=short -p no:cacheprovider -k "packed or field" > gpurun_out/pytest_r2v36.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v36.log
timeout 1500 python bench.py --no-configs --no-slab --no-pipeline-pass > gpurun_out/bench_r2v36.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v36.log
timeout 1500 python bench.py --no-configs --no-slab --no-pipeline-pass > gpurun_out/bench_r2v36b.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v36b.log
