mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_v15.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_v15.log
for S in stream level; do
timeout 300 python bench.py --steps 5 --warmup 3 --schedule $S --no-cpu-baseline --no-queries > gpurun_out/bench_v15_$S.jsonl 2>gpurun_out/bench_v15_$S.err; echo b$S=$?
done
timeout 300 python tools/qbench.py tf32x3 1 > gpurun_out/qb15_tf32x3.json 2>&1; echo q=$?
timeout 300 python tools/qbench.py bf16 1 > gpurun_out/qb15_bf16.json 2>&1; echo q=$?
