# r02chk: the sketch / first-sweep cap on large single-row problems; the whole non-C5 suite with the sketch forced on small problems
set -x
O=gpurun_out/r02chk
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "sketched" --durations=4 > $O/pytest_sketched.txt 2>&1; echo "rc=$?" >> $O/pytest_sketched.txt
TOPT_B200_SKETCH_MIN_N=1 timeout 1200 python -m pytest tests/ -q -m gpu --timeout 300 -k "not c5 and not strict" > $O/pytest_forced.txt 2>&1; echo "rc=$?" >> $O/pytest_forced.txt
TOPT_B200_SKETCH_MIN_N=1 TOPT_B200_FUSED_SWEEP=1 timeout 1200 python -m pytest tests/ -q -m gpu --timeout 300 -k "not c5 and not strict" > $O/pytest_forced_fused.txt 2>&1; echo "rc=$?" >> $O/pytest_forced_fused.txt
echo done
