timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_exact.py -q -x -k "exact" > gpurun_out/r02w_pytest.log 2>&1
echo "pytest rc=$?"; tail -n 4 gpurun_out/r02w_pytest.log
python -c "
import sys; sys.path.insert(0,'.')
import json, bench
print(json.dumps(bench.query_microbench('exact')))
" > gpurun_out/r02w_qbench.log 2>&1; tail -n 2 gpurun_out/r02w_qbench.log | cut -c1-1500
