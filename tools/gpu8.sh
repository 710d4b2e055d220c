timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r2v8.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r2v8.log
timeout 1200 python bench.py --workload c4 > gpurun_out/bench_c4_r2v8.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_r2v8.log
