timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_step.py --trace C4 2>&1 | cut -c1-130
timeout 300 python tools/prof_step.py --trace C2 2>&1 | cut -c1-130 | tail -3
timeout 600 python tools/c4_debug.py C4 4 2>&1 | grep -E "path|normwise|y abs|mask"
