mkdir -p gpurun_out
PYTHONPATH=. timeout 200 python tools/dbg_stream.py b 4 40 > gpurun_out/dbg6.log 2>&1; echo dbg6=$?
tail -6 gpurun_out/dbg6.log
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -k "stream" > gpurun_out/pytest_v8_stream.log 2>&1; echo pytest_stream=$?
tail -15 gpurun_out/pytest_v8_stream.log
timeout 300 python bench.py --steps 5 --warmup 3 --schedule stream --no-cpu-baseline --no-queries > gpurun_out/bench_v8_stream.jsonl 2>gpurun_out/bench_v8_stream.err; echo bs=$?
tail -3 gpurun_out/bench_v8_stream.err
