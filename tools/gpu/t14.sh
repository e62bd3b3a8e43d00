# 4 GPUs: multi-GPU tests, 512^3 bench at N=2 and 4, 256^3 strong scaling with comm columns, 1024^3 HIT
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rf > gpurun_out/t14_multi.log 2>&1
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus $N --steps 10 --warmup 3 --no-cpu > gpurun_out/t14_bench_n$N.json 2> gpurun_out/t14_bench_n$N.err
done
timeout 900 python -m paper_2211_16718_b200 scale --set n=256 --set scheme=rk4 --set cfl=0.4 --set mu=0.006 --ranks 1,2,4 --steps 10 > gpurun_out/t14_scale256.txt 2> gpurun_out/t14_scale256.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 \
  tools/big_decomp.py --grid 1024 --steps 100 --warmup 3 --cfl 0.3 > gpurun_out/t14_big1024.json 2> gpurun_out/t14_big1024.err
