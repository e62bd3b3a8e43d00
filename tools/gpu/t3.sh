timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_hit.py tests/test_gpu_parity.py -q -rf > gpurun_out/t3_pytest.log 2>&1
python tools/prof_step.py --n 256 --steps 1 --warmup 1 > gpurun_out/t3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -s 12 -c 3 -o gpurun_out/t3_sweeps python tools/prof_step.py --n 256 --steps 1 --warmup 1 > gpurun_out/t3_ncu.log 2>&1
