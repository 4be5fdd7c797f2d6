A="tools/plan_1_ph1.bin tools/tot_1_ph1.bin tools/plan_2_ph2.bin tools/tot_2_ph2.bin tools/plan_3_ph2.bin tools/tot_3_ph2.bin tools/plan_4_ph2.bin tools/tot_4_ph2.bin tools/plan_5_ph2.bin tools/tot_5_ph2.bin"
echo warp; ./tools/ctlbench $A
echo scalar; CTL_SCALAR=1 ./tools/ctlbench $A
