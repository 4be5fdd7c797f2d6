# r02m: ncu evidence on the committed code: k_step full sets (C5 headline, C3, C4, C2) + launch list of the default bench command
set -x
O=gpurun_out/r02m
mkdir -p $O
for cs in "C5 5" "C3 3" "C4 4" "C2 2"; do
  set -- $cs
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o /tmp/ncu_$1 python tools/prof_step.py --config $1 --seed $2 --steps 3 > $O/ncu_$1.log 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
echo done
