set -x
python bench.py --precision exact --no-queries --twopass-n 0 --no-cpu-baseline --steps 5 --warmup 3 --out gpurun_out/r02a_b_exact.json > gpurun_out/r02a_b_exact.log 2>&1
python bench.py --precision tf32x3 --no-queries --twopass-n 0 --no-cpu-baseline --steps 5 --warmup 3 --out gpurun_out/r02a_b_tf32x3.json > gpurun_out/r02a_b_tf32x3.log 2>&1
python bench.py --config e --e-total 296 --precision exact --no-cpu-baseline --steps 2 --warmup 1 --out gpurun_out/r02a_e_exact.json > gpurun_out/r02a_e_exact.log 2>&1
python bench.py --config e --e-total 296 --precision tf32x3 --no-cpu-baseline --steps 2 --warmup 1 --out gpurun_out/r02a_e_tf32x3.json > gpurun_out/r02a_e_tf32x3.log 2>&1
tail -3 gpurun_out/*.log
