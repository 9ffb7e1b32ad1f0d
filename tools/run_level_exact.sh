set -u
timeout 1200 python -m pytest "tests/test_gpu_fullsize.py::test_full_size_tf32x3_stream_vs_oracle" -q -s 2>&1 | grep "full length tf32x3\|passed\|failed" > gpurun_out/tf32_tests.log
