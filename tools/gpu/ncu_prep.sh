timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 72 -c 1 -o gpurun_out/pb_prep2 -f ./tools/passbench > gpurun_out/ncu_pb2.log 2>&1; echo ncu2 $?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 95 -c 1 -o gpurun_out/pb_step2 -f ./tools/passbench > gpurun_out/ncu_pb3.log 2>&1; echo ncu3 $?
