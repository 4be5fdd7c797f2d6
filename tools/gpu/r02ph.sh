set -x
O=gpurun_out/r02ph
mkdir -p $O
for c in C3 C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_pattern.py tests/test_gpu_parity.py tests/test_gpu_full.py -q --timeout 300 -k "not c5" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
