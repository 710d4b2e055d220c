bash tools/gpu20.sh
timeout 1200 python bench.py --no-slab --no-configs > gpurun_out/bench_r2v27.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v27.log
