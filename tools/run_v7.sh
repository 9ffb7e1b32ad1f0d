mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k "stream" > gpurun_out/pytest_v7_stream.log 2>&1; echo pytest_stream=$?
tail -15 gpurun_out/pytest_v7_stream.log
timeout 300 python bench.py --steps 5 --warmup 3 --schedule stream --no-cpu-baseline --no-queries > gpurun_out/bench_v7_stream.jsonl 2>gpurun_out/bench_v7_stream.err; echo bs=$?
tail -3 gpurun_out/bench_v7_stream.err
