CMD="python tools/qbench.py tf32x3 1"
$CMD > gpurun_out/qbench_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_advance_tc|k_word_logprob" -c 2 -o gpurun_out/prof_q $CMD > gpurun_out/ncu_q.log 2>&1
echo rc=$?
for p in bf16 tf32; do python tools/qbench.py $p 5 > gpurun_out/qbench_$p.log 2>&1; done
