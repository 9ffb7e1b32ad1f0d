set -u
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/all_tests.log
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.'); import bench
r = bench.beam_sweep('exact', beams=(8, 16, 32, 64), reps=2)
print(json.dumps(r))" > gpurun_out/sweep_auto.json 2> gpurun_out/sweep_auto.err
