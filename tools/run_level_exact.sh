# EXACT checks: full GPU suite, fat variant, a config-e solo line with phases
set -u
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/lx_tests.log
rm -f gpurun_out/fat_probe.jsonl
timeout 600 python tools/fat_probe.py 4 300 exact level >> gpurun_out/fat_probe.jsonl 2>> gpurun_out/fat_probe.err
timeout 300 python bench.py --e-total 592 --e-batch 148 --schedule stream1 --no-queries --no-wide --no-cpu-baseline --steps 2 --warmup 3 --out gpurun_out/solo_e148.json > gpurun_out/solo_e148.log 2>&1
