# full GPU suite + default bench line + reference arm (what the driver runs at round end)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/full_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -n 3 gpurun_out/full_pytest_gpu.log
python bench.py --steps 10 --warmup 3 --out gpurun_out/full_bench.json > gpurun_out/full_bench.log 2>&1
echo "bench rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 --out gpurun_out/full_ref.json > gpurun_out/full_ref.log 2>&1
echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1
echo "smoke rc=$?"; tail -n 2 gpurun_out/full_smoke.log
