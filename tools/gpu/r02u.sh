set -x
O=gpurun_out/r02u
mkdir -p $O
for c in C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_${c}.txt 2>&1; done
timeout 300 python -m pytest tests/test_gpu_pattern.py tests/test_gpu_parity.py -q --timeout 200 > $O/pytest_pattern.txt 2>&1; echo "rc=$?" >> $O/pytest_pattern.txt
