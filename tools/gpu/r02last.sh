# r02last: final code (L2 line prefetch in the pattern PREP and the large sweeps): traces, GPU suite, smoke, bench lines
set -x
O=gpurun_out/r02last
mkdir -p $O
for c in C2 C3 C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
for c in C1 C2 C3 C4 C4p; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1800 python -m pytest tests/ -q -m gpu --timeout 900 --durations=5 -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o /tmp/ncu_C5 python tools/prof_step.py --config C5 --seed 5 --steps 3 > $O/ncu_C5.log 2>&1
ncu -i /tmp/ncu_C5.ncu-rep --page raw --csv > $O/ncu_C5_raw.csv 2>&1
echo done
