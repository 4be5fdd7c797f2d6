set -x
O=gpurun_out/r02h
mkdir -p $O
timeout 600 python tools/strict_check.py > $O/strict.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_lockstep.py -q -k "not c5" > $O/pytest.txt 2>&1
for c in C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
