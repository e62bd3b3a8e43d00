timeout 600 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_parity.py tests/test_gpu_cabi.py -q -rf > gpurun_out/t17_pytest.log 2>&1
timeout 600 python tools/gpu/flux_probe.py 512 > gpurun_out/t17_flux.json 2> gpurun_out/t17_flux.err
