# tools/big_decomp.py across sizes / rank counts / halo paths / CFL (diagnosis matrix)
p=29600
run() {  # label nproc env args...
  local label=$1 np=$2 envs=$3; shift 3
  p=$((p+1))
  env $envs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port $p tools/big_decomp.py "$@" > gpurun_out/bm_$label.log 2>&1
  echo "$label rc=$? $(grep -h '^{' gpurun_out/bm_$label.log | tail -1) $(grep -h -m1 'StepError' gpurun_out/bm_$label.log | cut -c1-200)" >> gpurun_out/bm.txt
}
rm -f gpurun_out/bm.txt
run s1024n4 4 HD_PEER=1 --grid 1024 --steps 100 --cfl 0.3
run s1024n4cfl4 4 HD_PEER=1 --grid 1024 --steps 100 --cfl 0.4
run s1024n4nccl 4 HD_PEER=0 --grid 1024 --steps 20 --cfl 0.3
