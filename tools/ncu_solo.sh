# ncu of the one-CTA-per-stream EXACT kernel at config e (148 utterances x 300 frames = one bench batch)
# plus the launch list of a short default bench run
set -u
python tools/decode_once.py e 148 300 exact > gpurun_out/solo_once.json 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_decode_solo -c 1 -o gpurun_out/solo_full -f \
    python tools/decode_once.py e 148 300 exact > gpurun_out/solo_ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/solo_launches.csv \
    python bench.py --steps 2 --warmup 3 --e-total 592 --no-queries --no-cpu-baseline > gpurun_out/solo_ncu_launch.log 2>&1
