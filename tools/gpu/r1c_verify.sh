set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_c.log 2>&1; tail -c 2500 gpurun_out/bench_c.log
timeout 300 python tools/prof_step.py --trace > gpurun_out/trace_c.log 2>&1; tail -20 gpurun_out/trace_c.log
