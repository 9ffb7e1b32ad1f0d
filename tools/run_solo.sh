# EXACT parity tests, then config-e lines (solo kernel, the cluster kernel) and config b
set -u
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -5 > gpurun_out/solo_tests.log
timeout 300 python bench.py --e-total 592 --e-batch 148 --schedule stream1 --no-queries --no-cpu-baseline --steps 2 --warmup 3 --out gpurun_out/solo_e148.json > gpurun_out/solo_e148.log 2>&1
timeout 300 python bench.py --e-total 592 --e-batch 74 --schedule stream --no-queries --no-cpu-baseline --steps 2 --warmup 3 --out gpurun_out/solo_e74.json > gpurun_out/solo_e74.log 2>&1
timeout 300 python bench.py --config b --no-queries --twopass-n 0 --no-cpu-baseline --steps 3 --warmup 3 --out gpurun_out/solo_b.json > gpurun_out/solo_b.log 2>&1
