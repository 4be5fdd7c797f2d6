for c in C1 C2 C3 C4 C4p; do
  timeout 600 python bench.py --config $c --cpu-budget 5 > gpurun_out/bench_$c.log 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],3), 'cpu', round(d['cpu_baseline']['ms_per_step'],1), d['clocks']['reasons'])" || tail -3 gpurun_out/bench_$c.err
done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --cpu-budget 5 > gpurun_out/bench_C5.log 2> gpurun_out/bench_C5.err; tail -1 gpurun_out/bench_C5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', round(d['cpu_baseline']['ms_per_step'],1))"
for c in C2 C3 C4; do timeout 120 python tools/prof_step.py --trace $c > gpurun_out/r01e_trace_$c.txt 2>&1; done
timeout 600 python tools/c5_probe.py 512 --trace > gpurun_out/r01e_trace_C5.txt 2>&1
