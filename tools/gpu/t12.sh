export CUDA_LAUNCH_BLOCKING=1
for c in tma_ens tma; do timeout 120 python tools/gpu/tma_probe.py $c > gpurun_out/t12_$c.log 2>&1; echo "$c rc=$?" >> gpurun_out/t12_summary.log; done
unset CUDA_LAUNCH_BLOCKING
grep -q "rc=0" gpurun_out/t12_summary.log && timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/t12_pytest.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/t12_bench.json 2> gpurun_out/t12_bench.err
