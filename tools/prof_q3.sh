CMD="python tools/qbench.py tf32x3 1"
$CMD > gpurun_out/qb3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_advance_tc" -c 1 -o gpurun_out/prof_q3 $CMD > gpurun_out/ncu_q3.log 2>&1
echo rc=$?
