bash tools/gpu/iter.sh
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 3 -c 1 -o gpurun_out/pb_sweep -f ./tools/passbench > gpurun_out/ncu_pb1.log 2>&1; echo ncu1 $?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 72 -c 1 -o gpurun_out/pb_prep -f ./tools/passbench > gpurun_out/ncu_pb2.log 2>&1; echo ncu2 $?
