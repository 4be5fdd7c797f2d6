# r02t: pattern PREP (two sweeps, negated rows verified) + sketch from 32M elements
set -x
O=gpurun_out/r02t
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_pattern.py -q --timeout 200 > $O/pytest_pattern.txt 2>&1; echo "rc=$?" >> $O/pytest_pattern.txt
for c in C4 C5; do
  timeout 300 python tools/prof_step.py --trace $c > $O/trace_${c}.txt 2>&1
  TOPT_B200_PAT_HINT=0 timeout 300 python tools/prof_step.py --trace $c > $O/trace_${c}_nohint.txt 2>&1
done
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -k "not c5" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
echo done
