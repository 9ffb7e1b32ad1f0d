./tools/certify_micro > gpurun_out/certify.txt 2>&1
