# Fat variant (breadth 16, beam 64): full-length decodes per precision / schedule,
# then the level schedule's launch list (kernel shares) on a short run
set -u
rm -f gpurun_out/fat_probe.jsonl
for cfg in "exact level" "exact stream1" "exact stream"; do
  timeout 600 python tools/fat_probe.py 4 300 $cfg >> gpurun_out/fat_probe.jsonl 2>> gpurun_out/fat_probe.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fat_launches.csv \
  python tools/fat_probe.py 4 40 exact level > gpurun_out/fat_ncu.log 2>&1
