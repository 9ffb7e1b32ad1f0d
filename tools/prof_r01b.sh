CMD="python bench.py --steps 2 --warmup 1 --frames 30 --no-cpu-baseline --precision tf32x3"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hs_prim|k_advance_tc|k_expand|k_assign" -s 80 -c 4 -o gpurun_out/prof_r01b $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
