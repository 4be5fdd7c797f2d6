# ncu --set full of k_step on the final r01f code (exported to csv, reports deleted)
set -x
O=gpurun_out/r01f_ncu
mkdir -p $O
for cs in "C2 2" "C4 4"; do
  set -- $cs
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o /tmp/ncu_$1 python tools/prof_step.py --config $1 --seed $2 --steps 3 > $O/ncu_$1.log 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>&1
done
TOPT_B200_STREAM=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
echo done
