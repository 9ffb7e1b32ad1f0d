timeout 300 python bench.py --e-total 592 --e-batch 148 --schedule stream1 --no-queries --no-cpu-baseline --steps 2 --warmup 3 --out gpurun_out/solo_e148.json > gpurun_out/solo_e148.log 2>&1
