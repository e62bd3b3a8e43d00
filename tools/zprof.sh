# cost attribution of the fused z sweep (profiling switches, see hd_sweep.cu)
i=0
for cfg in "X=0" "HD_PROFILE_NO_DZ=1" "HD_PROFILE_NO_PRIMS=1" "HD_PROFILE_NO_DZ=1 HD_PROFILE_NO_PRIMS=1"; do
  env $cfg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"sweep_kernel" --csv --log-file gpurun_out/zprof_$i.csv python tools/prof_step.py --n 512 --steps 1 --warmup 1 > /dev/null 2>&1
  echo "$cfg" > gpurun_out/zprof_$i.cfg
  i=$((i+1))
done
