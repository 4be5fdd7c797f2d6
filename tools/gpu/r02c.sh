set -x
O=gpurun_out/r02c
mkdir -p $O
timeout 900 python tools/strict_check.py --c4 > $O/strict.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_strict.py -x -q -k "not c5" > $O/pytest_strict.txt 2>&1
