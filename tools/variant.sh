#!/bin/bash
# Build a library variant with extra -D flags on the box-solve units into
# tmp_variants/NAME.so (the other units from build/obj of the last build).
# Usage (build box, repo root): bash tools/variant.sh NAME "-DFOO=1 -DBAR=2"
NAME=$1; FLAGS=$2
mkdir -p tmp_variants build/var_$NAME
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
C=paper_2404_14864_b200/csrc
pids=""
for u in box_dir_f64 box_dir_c128; do
  nvcc $F $FLAGS -c -o build/var_$NAME/$u.o $C/$u.cu & pids="$pids $!"
done
for p in $pids; do wait $p || exit 1; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tmp_variants/$NAME.so \
  build/obj/kfbi_b200.o build/var_$NAME/box_dir_f64.o build/var_$NAME/box_dir_c128.o \
  build/obj/box_neu_f64.o build/obj/box_neu_c128.o && echo "built tmp_variants/$NAME.so"
