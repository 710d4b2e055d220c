SKIP_BOX=1 TEST_TIMEOUT=1500 PYTEST_ARGS="--tb=short" BENCH_ARGS="--steps 20 --warmup 3" bash tools/gpu_r2.sh r2v3
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_r2v3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_r2v3.log
