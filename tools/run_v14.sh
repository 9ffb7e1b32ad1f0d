mkdir -p gpurun_out
PYTHONPATH=. timeout 200 python tools/dbg_stream.py b 4 40 > gpurun_out/dbg14.log 2>&1; echo dbg=$?
tail -6 gpurun_out/dbg14.log
timeout 300 python bench.py --steps 5 --warmup 3 --schedule stream --no-cpu-baseline --no-queries > gpurun_out/bench_v14.jsonl 2>gpurun_out/bench_v14.err; echo b=$?
