#!/bin/bash
# A/B box-solve timing + accuracy of library variants in tmp_variants/.
# Usage (GPU box, repo root): bash tools/ab_box.sh "sizes" libA.so libB.so ...
SIZES=$1; shift
mkdir -p gpurun_out
cp paper_2404_14864_b200/libkfbi_b200.so /tmp/lib_orig.so
for v in "$@"; do
  cp tmp_variants/$v paper_2404_14864_b200/libkfbi_b200.so
  echo "== $v"
  timeout 600 python tools/check_box.py $SIZES 2>&1 | tail -20
done
cp /tmp/lib_orig.so paper_2404_14864_b200/libkfbi_b200.so
