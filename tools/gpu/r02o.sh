# r02o: after the controller phase-read race fix: optimizer drop-in, m = 0 direction jobs, whole GPU suite (C5 tests last, separately timed), traces
set -x
O=gpurun_out/r02o
mkdir -p $O
for n in 6144 2048 6000; do TOPT_B200_PROGRESS=1 timeout 20 python tools/gpu/pydir.py $n > $O/py_$n.txt 2>&1; echo rc=$? >> $O/py_$n.txt; done
timeout 30 stdbuf -o0 -e0 ./tests/cpp/optimizer_ours > $O/opt.txt 2>&1; echo rc=$? >> $O/opt.txt
TOPT_B200_PARITY=strict timeout 30 stdbuf -o0 -e0 ./tests/cpp/optimizer_ours > $O/opt_strict.txt 2>&1; echo rc=$? >> $O/opt_strict.txt
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 200 --durations=10 -k "not c5" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 900 --durations=10 -k "c5" > $O/pytest_c5.txt 2>&1; echo "rc=$?" >> $O/pytest_c5.txt
for c in C2 C3; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
echo done
