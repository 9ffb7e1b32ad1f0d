timeout 600 python -m pytest tests/test_gpu_exact.py -x -q 2>&1 | tail -3
python bench.py --precision exact --no-queries --twopass-n 0 --no-cpu-baseline --steps 5 --warmup 3 --out gpurun_out/r02e_b_exact.json > gpurun_out/r02e_b_exact.log 2>&1
python bench.py --config e --e-total 296 --precision exact --no-cpu-baseline --steps 2 --warmup 1 --out gpurun_out/r02e_e_exact.json > gpurun_out/r02e_e_exact.log 2>&1
tail -n 3 gpurun_out/r02e_b_exact.log | cut -c1-300
python tools/decode_once.py b 64 100 exact > gpurun_out/r02e_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_decode_streams -c 1 -o gpurun_out/r02e_exact python tools/decode_once.py b 64 100 exact > gpurun_out/r02e_ncu.log 2>&1
