# EXACT parity tests, then a config-e line of the one-CTA kernel (592 utterances, 148-stream batches)
set -u
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q 2>&1 | tail -5 > gpurun_out/solo_tests.log
timeout 300 python bench.py --e-total 592 --e-batch 148 --schedule stream1 --no-queries --no-wide --no-cpu-baseline --steps 2 --warmup 3 --out gpurun_out/solo_e148.json > gpurun_out/solo_e148.log 2>&1
