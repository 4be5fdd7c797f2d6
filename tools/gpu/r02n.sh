# r02n: diagnose the hung drop-in strict test; fused vs per-row sweep traces; structured trace; fast GPU suite with per-test timeout
set -x
O=gpurun_out/r02n
mkdir -p $O
timeout 60 ./tests/cpp/optimizer_ours > $O/opt.txt 2>&1; echo rc=$? >> $O/opt.txt
TOPT_B200_PARITY=strict timeout 60 ./tests/cpp/optimizer_ours > $O/opt_strict.txt 2>&1; echo rc=$? >> $O/opt_strict.txt
TOPT_B200_FUSED_SWEEP=0 TOPT_B200_PARITY=strict timeout 60 ./tests/cpp/optimizer_ours > $O/opt_strict_nofuse.txt 2>&1; echo rc=$? >> $O/opt_strict_nofuse.txt
for c in C4 C5; do
  timeout 300 python tools/prof_step.py --trace $c > $O/trace_${c}_fused.txt 2>&1
  TOPT_B200_FUSED_SWEEP=0 timeout 300 python tools/prof_step.py --trace $c > $O/trace_${c}_perrow.txt 2>&1
  timeout 300 python tools/prof_step.py --trace --structured $c > $O/trace_${c}_structured.txt 2>&1
done
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 150 --durations=25 --deselect tests/test_dropin_cpp.py::test_optimizer_dropin_strict_matches_oracle -k "not c5" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
echo done
