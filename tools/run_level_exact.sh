# EXACT level schedule checks: parity (exact / big-beam / fat) and the config-e schedule comparison
set -u
timeout 1500 python -m pytest tests/test_gpu_exact.py tests/test_gpu_bigbeam.py tests/test_gpu_decode.py "tests/test_gpu_fullsize.py::test_fat_variant_vs_oracle" "tests/test_gpu_fullsize.py::test_fat_variant_full_length_exact_modes_agree" -x -q 2>&1 | tail -5 > gpurun_out/lx_tests.log
rm -f gpurun_out/fat_probe.jsonl
timeout 600 python tools/fat_probe.py 4 300 exact level >> gpurun_out/fat_probe.jsonl 2>> gpurun_out/fat_probe.err
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.'); import bench
print(json.dumps(bench.fat_variant('exact')))
print(json.dumps(bench.beam_sweep('exact', beams=(32, 64), reps=2)))" > gpurun_out/lx_extras.json 2>> gpurun_out/fat_probe.err
