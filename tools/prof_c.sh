# ncu --set full (with source) of one config-c stream-kernel launch (H=512, V=64k, 64 streams)
mkdir -p gpurun_out /tmp/rep
TAG=${1:-r01l}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_streams --launch-skip 1 -c 1 -o /tmp/rep/${TAG}_c python tools/phases_c.py c 64 > gpurun_out/${TAG}_ncu_c.log 2>&1; echo full=$?
ncu -i /tmp/rep/${TAG}_c.ncu-rep --page raw --csv > gpurun_out/${TAG}_c_raw.csv 2>/dev/null
ncu -i /tmp/rep/${TAG}_c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_c_src.csv 2>/dev/null
ls -la gpurun_out | grep ${TAG}
