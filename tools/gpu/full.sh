date
timeout 900 python -m pytest tests/test_gpu_full.py -x -q -s 2>&1 | tail -15; echo rc=$?
date
