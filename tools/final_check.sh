# Round-end check on one 4-GPU box: GPU test suite, bench at N = 1, 2, 4 and the reference arm -> gpurun_out/final_*
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final_tests.log
python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/final_n2.json 2> gpurun_out/final_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/final_n4.json 2> gpurun_out/final_n4.err
python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
