set -x
python bench.py > gpurun_out/bench_r1b.log 2>&1; tail -c 3000 gpurun_out/bench_r1b.log
python bench.py --steps 3 --warmup 3 --cpu-budget 0.5 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 3 --warmup 3 --cpu-budget 0.5 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_step.py --steps 3 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/prof_r1b python tools/prof_step.py --steps 3 > gpurun_out/ncu_full_r1b.log 2>&1
python tools/prof_step.py --trace > gpurun_out/trace_r1b.log 2>&1
ls -la gpurun_out/ | tail -5
