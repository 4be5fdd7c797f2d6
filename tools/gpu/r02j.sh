set -x
O=gpurun_out/r02j
mkdir -p $O
TOPT_B200_PARITY=strict ./tests/cpp/optimizer_ours > $O/opt_strict.txt 2>&1; echo rc=$? >> $O/opt_strict.txt
./tests/cpp/optimizer_ours > $O/opt.txt 2>&1; echo rc=$? >> $O/opt.txt
timeout 900 python -m pytest tests/test_gpu_fea.py tests/test_gpu_upstream.py -q > $O/pytest.txt 2>&1
for c in C5; do timeout 300 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
