#!/bin/bash
# Build timing-experiment variants of the native library (tools only, never shipped):
#   tools/exp_variants.sh NAME "-DFLAG ..."   -> paper_2501_08582_b200/_native/exp/NAME.so
set -e
cd "$(dirname "$0")/.."
OUT=paper_2501_08582_b200/_native/exp/$1
mkdir -p "$OUT"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -Iinclude $2"
for s in lors_capi lors_simt lors_tc lors_decoder; do
  nvcc $F -c paper_2501_08582_b200/csrc/$s.cu -o $OUT/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/liblors_b200.so $OUT/*.o
echo $OUT/liblors_b200.so
