# NVLink bytes moved by a 2-GPU 512^3 march (z slabs, peer-store halo): NVML link
# counters before and after, and the run's JSON line (tools/gpu/nvlink_probe.sh OUTDIR)
out=${1:-gpurun_out}
python tools/gpu/nvlink_counters.py > $out/nvlink_before.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 \
  bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu --no-e2e > $out/nvlink_bench_n2.json 2> $out/nvlink_bench_n2.err
python tools/gpu/nvlink_counters.py > $out/nvlink_after.json 2>&1
