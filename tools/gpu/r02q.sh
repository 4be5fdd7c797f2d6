# r02q: pipelined fused sweep + 4-pass sketch
set -x
O=gpurun_out/r02q
mkdir -p $O
for c in C4 C5; do
  for f in 0 1; do
    TOPT_B200_FUSED_SWEEP=$f timeout 300 python tools/prof_step.py --trace $c > $O/trace_${c}_f${f}.txt 2>&1
  done
done
TOPT_B200_FUSED_SWEEP=1 TOPT_B200_SKETCH_MIN_N=0 timeout 300 python tools/prof_step.py --trace C4 > $O/trace_C4_f1_nosketch.txt 2>&1
TOPT_B200_FUSED_SWEEP=1 TOPT_B200_SKETCH_MIN_N=1 timeout 900 python -m pytest tests/ -q -m gpu --timeout 200 -k "not c5 and not strict" -x > $O/pytest_forced.txt 2>&1; echo "rc=$?" >> $O/pytest_forced.txt
TOPT_B200_FUSED_SWEEP=1 timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_parity.py tests/test_gpu_api.py -q --timeout 300 -k "not c5" > $O/pytest_fused.txt 2>&1; echo "rc=$?" >> $O/pytest_fused.txt
echo done
