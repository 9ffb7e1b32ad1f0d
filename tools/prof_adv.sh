CMD="python tools/qbench.py tf32x3 1"
ncu --set full --clock-control none --import-source on -k regex:"k_advance_tc" -c 1 -o gpurun_out/prof_adv $CMD > gpurun_out/ncu_adv.log 2>&1
echo rc=$?
