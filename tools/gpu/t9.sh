timeout 300 python tools/gpu/tma_known_good.py > gpurun_out/t9.log 2>&1; echo "rc=$?" >> gpurun_out/t9.log
