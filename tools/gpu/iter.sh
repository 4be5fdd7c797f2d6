# quick iteration: GPU parity tests, per-pass trace, bench line
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python tools/prof_step.py --trace > gpurun_out/trace.log 2>&1; cut -c1-200 gpurun_out/trace.log | tail -12
timeout 300 python bench.py --cpu-budget 0.5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e_ms', d['e2e']['ms_per_step'], d['config'])"
if [ -x tools/passbench ]; then timeout 60 ./tools/passbench > gpurun_out/passbench.log 2>&1; cat gpurun_out/passbench.log; fi
