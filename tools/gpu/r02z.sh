# r02z: FEAS pass returns Newton's first evaluation: traces + the whole GPU suite (C5 strict stays opt-in)
set -x
O=gpurun_out/r02z
mkdir -p $O
for c in C4 C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
timeout 2400 python -m pytest tests/ -q -m gpu --timeout 900 --durations=8 -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
echo done
