#!/bin/bash
# Build libhd.so variants with different sweep register caps into build/variants/
set -e
cd "$(dirname "$0")/../paper_2211_16718_b200/csrc"
mkdir -p ../../build/variants
for mb in "$@"; do
  out=../../build/variants/mb$mb
  mkdir -p $out
  for f in hd_sweep hd_field hd_api; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DHD_SWEEP_MIN_BLOCKS=$mb -c $f.cu -o $out/$f.o &
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libhd.so $out/*.o -lcudart
done
