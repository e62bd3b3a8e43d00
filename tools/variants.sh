#!/bin/bash
# Time bench.py (5 steps, per-kernel timer) against libhd.so variants built by
# tools/build_variants.sh:  tools/variants.sh base gz3 gzw2 ...  -> gpurun_out/variants.txt
rm -f gpurun_out/variants.txt
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L="HD_LIB=build/variants/$v/libhd.so"; fi
  env $L python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2), {k:round(v['avg_ms'],3) for k,v in d['roofline']['kernels'].items()})" >> gpurun_out/variants.txt
done
