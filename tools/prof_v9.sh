mkdir -p gpurun_out /tmp/rep
CMD="python bench.py --steps 1 --warmup 1 --schedule stream --no-cpu-baseline --no-queries"
K=k_decode_streams
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip 1 -c 1 -o /tmp/rep/v19 $CMD > gpurun_out/ncu_v19.log 2>&1; echo ncu=$?
ncu -i /tmp/rep/v19.ncu-rep --page raw --csv > gpurun_out/v19_raw.csv 2>/dev/null
ncu -i /tmp/rep/v19.ncu-rep --page details --csv > gpurun_out/v19_details.csv 2>/dev/null
ncu -i /tmp/rep/v19.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/v19_src.csv 2>/dev/null
ls -la /tmp/rep gpurun_out/v9*
