timeout 1500 python -m pytest tests/test_gpu_ngram3.py tests/test_gpu_fullsize.py -q -x -k "ngram3 or exact or trigram or pinned or tf32x3_stream or fat" > gpurun_out/r02u_pytest.log 2>&1
echo "pytest rc=$?"
tail -n 5 gpurun_out/r02u_pytest.log
