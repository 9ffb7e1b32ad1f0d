mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --schedule stream --precision tf32 --no-cpu-baseline --no-queries > gpurun_out/bench_v12_tf32.jsonl 2>gpurun_out/bench_v12.err; echo b=$?
