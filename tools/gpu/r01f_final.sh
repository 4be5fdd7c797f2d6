# final r01f bench lines on the committed code
set -x
O=gpurun_out/r01f_final
mkdir -p $O
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in C2 C1 C3 C4 C4p C5; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for c in C2 C4 C5; do timeout 200 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
echo done
