mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --precision fp64 --schedule level --groups 4 --no-cpu-baseline --no-queries > gpurun_out/bench_fp64.jsonl 2> gpurun_out/bench_fp64.err; echo b=$?
