timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "staged" > gpurun_out/t19_pytest.log 2>&1
timeout 600 python tools/gpu/option_probe.py 512 X_STAGED 1,2 > gpurun_out/t19_probe.json 2> gpurun_out/t19_probe.err
