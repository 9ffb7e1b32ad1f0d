timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02t_pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -n 3 gpurun_out/r02t_pytest_gpu.log
python bench.py --steps 5 --warmup 3 --out gpurun_out/r02t_bench.json > gpurun_out/r02t_bench.log 2>&1
echo "bench rc=$?"
