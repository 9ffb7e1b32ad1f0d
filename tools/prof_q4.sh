CMD="python tools/qbench.py bf16 1"
$CMD > gpurun_out/qb4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_advance_tc" -c 1 -o gpurun_out/prof_q4 $CMD > gpurun_out/ncu_q4.log 2>&1
echo rc=$?
