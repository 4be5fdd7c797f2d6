# r02l: full -m gpu suite, smoke, all-config bench lines, reference arm, traces (committed code)
set -x
O=gpurun_out/r02l
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
for c in C1 C2 C3 C4 C4p; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 400 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for c in C2 C3 C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
echo done
