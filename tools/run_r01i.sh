# quick iteration: GPU tests + default bench line (with phase timers) + config-c phases
mkdir -p gpurun_out
TAG=${1:-r01i}
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --twopass-n 0 > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench=$?
timeout 600 python tools/phases_c.py > gpurun_out/${TAG}_phases_c.json 2> gpurun_out/${TAG}_phases_c.err; echo phc=$?
