set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v6.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_v6.log
timeout 300 python bench.py --steps 5 --warmup 3 --groups 1 --no-cpu-baseline --no-queries > gpurun_out/bench_v6_g1.jsonl 2>gpurun_out/bench_v6_g1.err; echo b1=$?
timeout 300 python bench.py --steps 5 --warmup 3 --groups 4 --no-cpu-baseline --no-queries > gpurun_out/bench_v6_g4.jsonl 2>gpurun_out/bench_v6_g4.err; echo b4=$?
timeout 300 python bench.py --steps 5 --warmup 3 --groups 4 --precision bf16 --no-cpu-baseline --no-queries > gpurun_out/bench_v6_bf16.jsonl 2>gpurun_out/bench_v6_bf16.err; echo bbf=$?
