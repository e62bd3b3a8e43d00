timeout 300 python bench.py --steps 6 --warmup 2 --no-cpu --no-e2e > gpurun_out/t13_bench.json 2> gpurun_out/t13_bench.err
python tools/prof_step.py --n 256 --steps 1 --warmup 1 > gpurun_out/t13_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep|gradflux" -s 16 -c 4 -o gpurun_out/t13_prof python tools/prof_step.py --n 256 --steps 1 --warmup 1 > gpurun_out/t13_ncu.log 2>&1
