#!/bin/bash
# ncu --set full of the column pass (and the row passes) at M = 4096 for the
# library variants given.  Usage (GPU box): bash tools/prof_tri.sh TAG libA.so ...
TAG=$1; shift
cp paper_2404_14864_b200/libkfbi_b200.so /tmp/lib_orig.so
for v in "$@"; do
  cp tmp_variants/$v paper_2404_14864_b200/libkfbi_b200.so
  for c in real complex; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cols_|rows_" -s 6 -c 3 \
      -o gpurun_out/prof_${TAG}_${v%.so}_$c -f python tools/prof_box.py 4096 3 $c > gpurun_out/prof_${TAG}_${v%.so}_$c.log 2>&1
    python tools/ncu_summary.py gpurun_out/prof_${TAG}_${v%.so}_$c.json gpurun_out/prof_${TAG}_${v%.so}_$c.ncu-rep > /dev/null 2>&1
  done
done
cp /tmp/lib_orig.so paper_2404_14864_b200/libkfbi_b200.so
