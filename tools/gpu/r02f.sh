set -x
O=gpurun_out/r02f
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_campaign.py tests/test_gpu_strict.py tests/test_gpu_full.py -q -k "not c5" > $O/pytest.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o /tmp/ncu_C5 python tools/prof_step.py --config C5 --seed 5 --steps 3 > $O/ncu_C5.log 2>&1
ncu -i /tmp/ncu_C5.ncu-rep --page raw --csv > $O/ncu_C5_raw.csv 2>&1
ncu -i /tmp/ncu_C5.ncu-rep --page source --csv --print-source sass > /tmp/src_C5.csv 2>&1
gzip -c /tmp/src_C5.csv > $O/ncu_C5_src.csv.gz
ncu -i /tmp/ncu_C5.ncu-rep --page source --csv --print-source cuda > /tmp/srcc_C5.csv 2>&1
gzip -c /tmp/srcc_C5.csv > $O/ncu_C5_srccuda.csv.gz
ls -la $O
