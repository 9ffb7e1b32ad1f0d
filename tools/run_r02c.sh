python tools/decode_once.py b 64 100 exact > gpurun_out/r02c_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_decode_streams -c 1 -o gpurun_out/r02c_exact python tools/decode_once.py b 64 100 exact > gpurun_out/r02c_ncu.log 2>&1
tail -2 gpurun_out/r02c_plain.log gpurun_out/r02c_ncu.log
