date
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --cpu-budget 5 > gpurun_out/bench_C5.log 2> gpurun_out/bench_C5.err; echo rc=$?
tail -1 gpurun_out/bench_C5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'e2e_ms', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline'], d['config'])"
tail -8 gpurun_out/bench_C5.err
date
