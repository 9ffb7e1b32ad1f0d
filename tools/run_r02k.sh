python bench.py --precision exact --no-queries --twopass-n 0 --no-cpu-baseline --steps 3 --warmup 3 --out gpurun_out/r02k_b_exact.json > gpurun_out/r02k_b_exact.log 2>&1
