#!/bin/bash
# ncu launch times of selected kernels for library variants in tmp_variants/.
# Usage (GPU box): bash tools/ncu_variant.sh "kernel regex" libA.so libB.so ...
RX=$1; shift
cp paper_2404_14864_b200/libkfbi_b200.so /tmp/lib_orig.so
for v in "$@"; do
  cp tmp_variants/$v paper_2404_14864_b200/libkfbi_b200.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
    -k regex:"$RX" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile > gpurun_out/ncuv_$v.csv 2>&1
  python - "$v" <<'PY'
import csv, sys, collections
v = sys.argv[1]
t = collections.defaultdict(list)
for r in csv.reader(open(f"gpurun_out/ncuv_{v}.csv")):
    if len(r) > 14 and r[12] == "gpu__time_duration.sum":
        t[r[4].split("(")[0][:50]].append(float(r[14]) / 1e3)
print(v, {k: [round(x, 1) for x in vals] for k, vals in t.items()})
PY
done
cp /tmp/lib_orig.so paper_2404_14864_b200/libkfbi_b200.so
