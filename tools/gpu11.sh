timeout 600 python -m pytest tests/test_gpu_gmres.py -q -s --tb=short -p no:cacheprovider > gpurun_out/pytest_gmres2.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r2v11.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r2v11.log
bash tools/sanitize.sh
