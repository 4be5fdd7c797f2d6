# prefetch check + launch list of the default bench command (streaming off under ncu:
# a serialised kernel cannot see the host's concurrent chunk copies)
set -x
O=gpurun_out/r01f_b
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in C1 C2; do timeout 300 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 200 python tools/prof_step.py --trace C2 > $O/trace_C2.txt 2>&1
TOPT_B200_STREAM=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
echo done
