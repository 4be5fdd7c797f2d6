# round-1 (session f) measurement set: bench lines, traces, launch list, ncu full of k_step.
# ncu reports are exported to csv on the box and deleted (gpurun_out/ must stay < 64 MiB).
set -x
O=gpurun_out/r01f
mkdir -p $O
for c in C1 C2 C3 C4 C4p C5; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for c in C2 C3 C4 C5; do timeout 200 python tools/prof_step.py --trace $c > $O/trace_$c.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
for cs in "C2 2" "C4 4"; do
  set -- $cs
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o /tmp/ncu_$1 python tools/prof_step.py --config $1 --seed $2 --steps 3 > $O/ncu_$1.log 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page source --csv --print-source sass > /tmp/src_$1.csv 2>&1
  gzip -c /tmp/src_$1.csv > $O/ncu_$1_src.csv.gz
done
du -sh $O
echo done
