timeout 1500 python bench.py --no-configs --no-slab > gpurun_out/bench_r2v61.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v61.log
