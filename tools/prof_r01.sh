set -x
CMD="python bench.py --steps 2 --warmup 1 --frames 30 --no-cpu-baseline --precision tf32x3"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"k_hs_prim|k_advance_tc|k_expand" -s 60 -c 3 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
