CMD="python tools/qbench.py tf32x3 1"
$CMD > gpurun_out/qb2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_advance_tc|k_word_logprob_ring" -c 2 -o gpurun_out/prof_q2 $CMD > gpurun_out/ncu_q2.log 2>&1
echo rc=$?
