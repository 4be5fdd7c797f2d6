for c in C1 C2 C3 C4 C4p C5; do
  timeout 900 python bench.py --config $c --cpu-budget 5 > gpurun_out/bench_$c.log 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'n', d['config']['n'], 'ms', round(d['ms_per_step'],4), 'Gvars/s', round(d['value']/1e9,3), 'frac', round(d['roofline']['frac'],4), 'e2e_ms', round(d['e2e']['ms_per_step'],3), 'cpu_ms', round(d['cpu_baseline']['ms_per_step'],1), 'cpu_n', d['cpu_baseline']['sample'][:60], d['config']['path'], d['config']['passes_per_step'], d['config']['sweeps_per_step'], d['clocks'])" || tail -3 gpurun_out/bench_$c.err
done
