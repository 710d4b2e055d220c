#!/bin/bash
# A/B the in-tree library against variants in tmp_variants/: bench each.
# Usage (GPU box, repo root): bash tools/ab.sh "bench args" libA.so libB.so ...
ARGS=$1; shift
mkdir -p gpurun_out
cp paper_2404_14864_b200/libkfbi_b200.so /tmp/lib_orig.so
for v in "$@"; do
  cp tmp_variants/$v paper_2404_14864_b200/libkfbi_b200.so
  timeout 600 python bench.py --no-cpu-baseline $ARGS > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/ab_{v}.log") if x.startswith("{")]
d = json.loads(l[-1]) if l else {}
print(v, d.get("value"), d.get("kernel_ms_per_bench_step"), {k: e["ms_per_step"] for k, e in d.get("per_equation", {}).items()})
PY
done
cp /tmp/lib_orig.so paper_2404_14864_b200/libkfbi_b200.so
