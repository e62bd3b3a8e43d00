timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/t16_bench.json 2> gpurun_out/t16_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/t16_ref.json 2> gpurun_out/t16_ref.err
python tools/prof_step.py --n 512 --steps 1 --warmup 1 > gpurun_out/t16_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t16_launches.csv python tools/prof_step.py --n 512 --steps 1 --warmup 1 > gpurun_out/t16_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|gradflux" -s 12 -c 3 -o gpurun_out/t16_prof python tools/prof_step.py --n 512 --steps 1 --warmup 1 > gpurun_out/t16_ncu.log 2>&1
