timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/t4_pytest.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/t4_bench.json 2> gpurun_out/t4_bench.err
