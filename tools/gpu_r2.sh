#!/bin/bash
# Round-2 GPU session: smoke, GPU tests, box-solve sizes for both column
# solvers, bench.  Usage (repo root, on the GPU box): bash tools/gpu_r2.sh TAG
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
fi
if [ "${SKIP_BOX:-0}" != "1" ]; then
  for c in tridiagonal dst; do
    KFBI_COLS=$c timeout 600 python tools/check_box.py ${BOX_SIZES:-256 1024 2048 4096 8192} > $OUT/check_box_${c}_$TAG.log 2>&1
  done
fi
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench_$TAG.log 2>&1; echo "rc=$?" >> $OUT/bench_$TAG.log
fi
