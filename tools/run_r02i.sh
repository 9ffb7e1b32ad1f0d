timeout 600 python -m pytest tests/test_gpu_exact.py -x -q 2>&1 | tail -3 > gpurun_out/r02i_tests.log
python bench.py --precision exact --no-queries --twopass-n 0 --no-cpu-baseline --steps 5 --warmup 3 --out gpurun_out/r02i_b_exact.json > gpurun_out/r02i_b_exact.log 2>&1
python bench.py --config e --e-total 296 --precision exact --no-cpu-baseline --steps 2 --warmup 1 --out gpurun_out/r02i_e_exact.json > gpurun_out/r02i_e_exact.log 2>&1
tail -n 3 gpurun_out/r02i_b_exact.log | cut -c1-300
