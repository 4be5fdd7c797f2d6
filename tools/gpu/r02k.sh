set -x
O=gpurun_out/r02k
mkdir -p $O
TOPT_B200_PARITY=strict ./tests/cpp/optimizer_ours > $O/opt_strict.txt 2>&1; echo rc=$? >> $O/opt_strict.txt
timeout 600 python tools/strict_check.py --c4 > $O/strict.txt 2>&1
timeout 1800 python -m pytest tests/ -q -m gpu -k "not c5" > $O/pytest.txt 2>&1
for c in C2 C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
