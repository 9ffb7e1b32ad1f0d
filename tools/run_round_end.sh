# round-end evidence: GPU suite, default bench line (+ extras), reference arm, smoke,
# ncu launch list of the default bench and a full capture of k_decode_solo,
# the fat variant's launch list (level schedule: k_expand_big / k_asg_*)
set -u
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/re_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -n 2 gpurun_out/re_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --out gpurun_out/re_bench.json > gpurun_out/re_bench.log 2>&1
echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 --out gpurun_out/re_ref.json > gpurun_out/re_ref.log 2>&1
echo "ref rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1
echo "smoke rc=$?"; tail -n 1 gpurun_out/re_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/re_launches.csv \
    python bench.py --steps 2 --warmup 3 --e-total 592 --no-queries --no-wide --no-cpu-baseline > gpurun_out/re_ncu_launch.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decode_solo -c 1 -o gpurun_out/re_solo_full -f \
    python tools/decode_once.py e 148 300 exact > gpurun_out/re_solo_ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/re_fat_launches.csv \
    python tools/fat_probe.py 4 300 exact level > gpurun_out/re_fat_ncu.log 2>&1
echo "fat launches rc=$?"
