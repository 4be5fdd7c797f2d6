# r02w: hybrid wide (per-lane) / lean (transposed) per-row sweep
set -x
O=gpurun_out/r02w
mkdir -p $O
for c in C2 C3 C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_${c}.txt 2>&1; done
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -k "not c5" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
TOPT_B200_SKETCH_MIN_N=1 timeout 900 python -m pytest tests/ -q -m gpu --timeout 200 -k "not c5 and not strict" -x > $O/pytest_forced.txt 2>&1; echo "rc=$?" >> $O/pytest_forced.txt
echo done
