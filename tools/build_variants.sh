#!/bin/bash
# Build libhd.so variants into build/variants/<name>/ ; each arg is name:DEFINES (comma-separated)
#   tools/build_variants.sh reg4:HD_SWEEP_MIN_BLOCKS=4 smem5:HD_SWEEP_SMEM_WINDOW=1,HD_SWEEP_MIN_BLOCKS=5
#   raw nvcc flags start with '-' ('@' stands for a space): cg:-Xptxas@-dlcm=cg
set -e
cd "$(dirname "$0")/../paper_2211_16718_b200/csrc"
for spec in "$@"; do
  name=${spec%%:*}
  defs=""
  IFS=',' read -ra kv <<< "${spec#*:}"
  for d in "${kv[@]}"; do
    if [[ "$d" == -* ]]; then defs="$defs ${d//@/ }"; else defs="$defs -D$d"; fi  # raw flag: '@' = space
  done
  out=../../build/variants/$name
  mkdir -p $out
  for f in hd_sweep hd_field hd_api hd_bench hd_peer hd_compat; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $defs -Xptxas -v -c $f.cu -o $out/$f.o 2> $out/$f.ptxas.log &
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libhd.so $out/*.o -lcudart
  rm -f $out/*.o  # only the .so travels to the GPU box (gpurun snapshot limit)
  echo "$name: $(grep -c spill $out/hd_sweep.ptxas.log) kernels, spills: $(grep 'spill' $out/hd_sweep.ptxas.log | grep -v ' 0 bytes spill stores' | wc -l)"
done
