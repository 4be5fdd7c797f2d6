# r02y: C5 against the reference golden (certified + strict), the new strict seeds, first-sweep candidate cap experiment
set -x
O=gpurun_out/r02y
mkdir -p $O
for k in 0 8 6; do
  TOPT_B200_FIRST_K=$k timeout 300 python tools/prof_step.py --trace C5 > $O/trace_C5_k$k.txt 2>&1
  TOPT_B200_FIRST_K=$k TOPT_B200_SKETCH_MIN_N=4194304 timeout 300 python tools/prof_step.py --trace C4 > $O/trace_C4_k$k.txt 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_full.py tests/test_gpu_strict.py -q --timeout 1100 --durations=8 -k "more_paths or certified" > $O/pytest_new.txt 2>&1; echo "rc=$?" >> $O/pytest_new.txt
timeout 2400 python -m pytest tests/test_gpu_strict.py -q --timeout 2300 --durations=4 -k "c5" > $O/pytest_c5_strict.txt 2>&1; echo "rc=$?" >> $O/pytest_c5_strict.txt
echo done
