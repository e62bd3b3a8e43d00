timeout 900 python tools/gpu/waves_probe.py 256x256x64,256x256x128,256x256x256,512x512x128,512x512x512 1,2,3,4,6,8 > gpurun_out/t15_waves.log 2>&1
