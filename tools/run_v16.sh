mkdir -p gpurun_out
PYTHONPATH=. timeout 200 python tools/dbg_stream.py b 4 40 > gpurun_out/dbg16.log 2>&1; echo dbg=$?
tail -4 gpurun_out/dbg16.log
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -k stream > gpurun_out/pytest_v16.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_v16.log
timeout 300 python bench.py --steps 5 --warmup 3 --schedule stream --no-cpu-baseline --no-queries > gpurun_out/bench_v16.jsonl 2>gpurun_out/bench_v16.err; echo b=$?
timeout 300 python tools/qbench.py tf32x3 1 > gpurun_out/qb16.json 2>&1; echo q=$?
