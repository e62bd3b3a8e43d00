# tools/big_decomp.py across sizes / rank counts / halo paths / CFL / block shapes (diagnosis matrix)
p=29600
run() {  # label nproc env args...
  local label=$1 np=$2 envs=$3; shift 3
  p=$((p+1))
  env $envs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port $p tools/big_decomp.py "$@" > gpurun_out/bm_$label.log 2>&1
  echo "$label rc=$? $(grep -h '^{' gpurun_out/bm_$label.log | tail -1) $(grep -h -m1 'StepError' gpurun_out/bm_$label.log | cut -c1-200)" >> gpurun_out/bm.txt
}
rm -f gpurun_out/bm.txt
run s512z256d114 4 HD_PEER=1 --grid 512 --nz 256 --steps 30 --cfl 0.4 --dims 1,1,4
run s512z256d122 4 HD_PEER=1 --grid 512 --nz 256 --steps 30 --cfl 0.4 --dims 1,2,2
run s512z256d212 4 HD_PEER=1 --grid 512 --nz 256 --steps 30 --cfl 0.4 --dims 2,1,2
