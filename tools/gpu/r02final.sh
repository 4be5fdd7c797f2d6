# r02final: evidence on the final round-2 code: traces, whole GPU suite, smoke, bench lines, reference arm, ncu
set -x
O=gpurun_out/r02final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
for c in C2 C3 C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
TOPT_B200_FIRST_K=4 timeout 300 python tools/prof_step.py --trace C5 > $O/trace_C5_k4.txt 2>&1
TOPT_B200_FIRST_K=4 timeout 300 python tools/prof_step.py --trace C4 > $O/trace_C4_k4.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu --timeout 900 --durations=8 -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 900 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
for c in C1 C2 C3 C4 C4p; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 400 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for cs in "C5 5" "C4 4"; do
  set -- $cs
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o /tmp/ncu_$1 python tools/prof_step.py --config $1 --seed $2 --steps 3 > $O/ncu_$1.log 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
echo done
