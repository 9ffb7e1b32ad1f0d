python bench.py --config b --no-queries --twopass-n 0 --no-cpu-baseline --steps 3 --warmup 3 --out gpurun_out/r02q_b.json > gpurun_out/r02q_b.log 2>&1
