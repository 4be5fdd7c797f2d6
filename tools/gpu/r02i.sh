set -x
O=gpurun_out/r02i
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fea.py tests/test_gpu_upstream.py tests/test_dropin_cpp.py tests/test_gpu_parity.py -q -x > $O/pytest.txt 2>&1
for c in C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
