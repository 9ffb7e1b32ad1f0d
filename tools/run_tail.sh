# a 512-utterance shard (the per-rank share at 8 GPUs): tail batch on its own decoder vs padded
set -u
timeout 600 python bench.py --e-total 512 --no-queries --no-wide --no-cpu-baseline --steps 3 --warmup 3 --out gpurun_out/tail_auto.json > gpurun_out/tail_auto.log 2>&1
timeout 600 python bench.py --e-total 512 --schedule stream1 --no-queries --no-wide --no-cpu-baseline --steps 3 --warmup 3 --out gpurun_out/tail_pad.json > gpurun_out/tail_pad.log 2>&1
