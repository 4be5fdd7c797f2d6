python -m pytest tests -m gpu -x -q -k "not full" 2>&1 | tail -3
python tools/e2e_probe.py 2>&1 | tail -4
TOPT_B200_STREAM=0 python tools/e2e_probe.py 2>&1 | tail -2
