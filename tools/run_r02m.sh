timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02m_pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -n 5 gpurun_out/r02m_pytest_gpu.log
