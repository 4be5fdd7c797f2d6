# round 2 first look: chain latency probe, C5 bench on the round-1 code, streaming under serialization
set -x
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 120 ./tools/chainbench > $O/chainbench.txt 2>&1
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
timeout 120 env CUDA_LAUNCH_BLOCKING=1 python -c "
import sys; sys.path.insert(0,'.')
import __graft_entry__ as g; g.smoke()" > $O/smoke_blocking.txt 2>&1
echo rc=$? >> $O/smoke_blocking.txt
nproc > $O/host.txt; lscpu | head -20 >> $O/host.txt; free -g >> $O/host.txt
