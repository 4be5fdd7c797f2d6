timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_step.py --trace C4 2>&1 | cut -c1-110
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 2 -c 1 -o gpurun_out/c4_kstep -f python tools/prof_step.py --config C4 --steps 3 > gpurun_out/ncu_c4.log 2>&1; echo ncu $?
