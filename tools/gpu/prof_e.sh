python tools/prof_step.py --steps 3 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/r01e_c2 -f python tools/prof_step.py --steps 3 > gpurun_out/ncu_full.log 2>&1; echo c2 $?
python tools/prof_step.py --config C4 --seed 4 --steps 3 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/r01e_c4 -f python tools/prof_step.py --config C4 --seed 4 --steps 3 > gpurun_out/ncu_full4.log 2>&1; echo c4 $?
python bench.py --steps 3 --warmup 3 --cpu-budget 0.5 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 40 --log-file gpurun_out/r01e_launches.csv python bench.py --steps 3 --warmup 3 --cpu-budget 0.5 > gpurun_out/ncu_launch.log 2>&1; echo launches $?
