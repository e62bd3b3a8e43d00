# 4-GPU bench with the NVLink peer-store halo vs the NCCL halo (HD_PEER=0): per-kernel times -> gpurun_out/mg.txt
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "decomposed or scale" > gpurun_out/multi.log 2>&1
p=29640
for cfg in "HD_PEER=1" "HD_PEER=0"; do
  p=$((p+1))
  env $cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 6 --warmup 2 --no-e2e --no-cpu > gpurun_out/mg_$p.log 2>&1
  tail -1 gpurun_out/mg_$p.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('$cfg', round(d['ms_per_step'],2), 'kern/step', round(sum(b['avg_ms']*b['launches'] for b in k.values())/d['steps'],2), {a:round(b['avg_ms'],3) for a,b in k.items()})" >> gpurun_out/mg.txt
done
