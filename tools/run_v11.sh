mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --schedule stream --no-cpu-baseline --no-queries > gpurun_out/bench_v11.jsonl 2>gpurun_out/bench_v11.err; echo b=$?
