for cfg in "fp64 level" "exact level" "exact stream" "tf32x3 stream"; do
  timeout 600 python tools/fat_probe.py 4 300 $cfg >> gpurun_out/fat_probe.jsonl 2>> gpurun_out/fat_probe.err
done
