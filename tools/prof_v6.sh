mkdir -p gpurun_out /tmp/rep
CMD="python bench.py --steps 1 --warmup 1 --groups 1 --no-cpu-baseline --no-queries --no-graph"
for K in k_advance_tc k_hs_prim_ring k_expand k_assign; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip 150 -c 1 -o /tmp/rep/v6_$K $CMD > gpurun_out/ncu_v6_$K.log 2>&1; echo $K=$?
ncu -i /tmp/rep/v6_$K.ncu-rep --page raw --csv > gpurun_out/v6_${K}_raw.csv 2>/dev/null
ncu -i /tmp/rep/v6_$K.ncu-rep --page details --csv > gpurun_out/v6_${K}_details.csv 2>/dev/null
ncu -i /tmp/rep/v6_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/v6_${K}_sass.csv 2>/dev/null
ls -la /tmp/rep
done
du -sh gpurun_out
