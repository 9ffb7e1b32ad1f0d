set -u
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | tail -15 > gpurun_out/mr_tests.log
