# one-CTA-per-stream EXACT kernel: parity tests, then config-e lines for several batch sizes
set -u
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q 2>&1 | tail -5 > gpurun_out/solo_tests.log
for B in 148 296 592; do
timeout 300 python bench.py --e-total 592 --e-batch $B --schedule stream1 --no-queries --no-cpu-baseline --steps 2 --warmup 3 --out gpurun_out/solo_e$B.json > gpurun_out/solo_e$B.log 2>&1
done
