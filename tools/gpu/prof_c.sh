set -x
python bench.py --steps 3 --warmup 3 --cpu-budget 0.5 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_launches.csv python bench.py --steps 3 --warmup 3 --cpu-budget 0.5 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_step.py --steps 3 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/r01c_c2 -f python tools/prof_step.py --steps 3 > gpurun_out/ncu_full.log 2>&1
python tools/prof_step.py --trace C2 > gpurun_out/r01c_trace_C2.txt 2>&1
python tools/prof_step.py --trace C4 > gpurun_out/r01c_trace_C4.txt 2>&1
python tools/prof_step.py --trace C3 > gpurun_out/r01c_trace_C3.txt 2>&1
python tools/c5_probe.py 512 --trace > gpurun_out/r01c_trace_C5.txt 2>&1
ls -la gpurun_out/ | tail -8
