set -x
O=gpurun_out/r02b
mkdir -p $O
timeout 900 python tools/strict_check.py --c4 > $O/strict.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -x -q > $O/pytest.txt 2>&1
