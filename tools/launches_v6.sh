mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_v6.csv python bench.py --steps 1 --warmup 1 --groups 1 --no-cpu-baseline --no-queries --no-graph > gpurun_out/ncu_v6.log 2>&1; echo ncu=$?
