python tools/xtile_check.py --n 128 --steps 3 > gpurun_out/xt_128.json 2>&1
python tools/xtile_check.py --n 512 --steps 3 > gpurun_out/xt_base.json 2>&1
for v in xt128m6 xt256m3 xt64m10; do HD_LIB=build/variants/$v/libhd.so python tools/xtile_check.py --n 512 --steps 3 > gpurun_out/xt_$v.json 2>&1; done
