timeout 300 python tools/gpu/power_probe.py 512 > gpurun_out/t18_power.log 2>&1
