python bench.py --e-total 296 --no-queries --no-cpu-baseline --steps 2 --warmup 1 --out gpurun_out/r02ab_e.json > gpurun_out/r02ab_e.log 2>&1
