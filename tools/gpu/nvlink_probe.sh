# NVLink bytes moved by a 2-GPU 512^3 march (z slabs, peer-store halo): the per-link
# data counters before and after, and the run's JSON line (tools/gpu/nvlink_probe.sh OUTDIR)
out=${1:-gpurun_out}
nvidia-smi nvlink -gt d > $out/nvlink_before.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 \
  bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu --no-e2e > $out/nvlink_bench_n2.json 2> $out/nvlink_bench_n2.err
nvidia-smi nvlink -gt d > $out/nvlink_after.txt 2>&1
nvidia-smi topo -m > $out/nvlink_topo.txt 2>&1
