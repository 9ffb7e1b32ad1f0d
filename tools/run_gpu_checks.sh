# GPU checks used while developing (run under gpurun): the EXACT parity tests,
# then a config-b and a short config-e bench line with the per-level phases.
set -u
timeout 600 python -m pytest tests/test_gpu_exact.py -x -q 2>&1 | tail -2 > gpurun_out/checks_tests.log
python bench.py --config b --no-queries --twopass-n 0 --no-cpu-baseline --steps 3 --warmup 3 --out gpurun_out/checks_b.json > gpurun_out/checks_b.log 2>&1
python bench.py --e-total 296 --no-queries --no-cpu-baseline --steps 2 --warmup 1 --out gpurun_out/checks_e.json > gpurun_out/checks_e.log 2>&1
