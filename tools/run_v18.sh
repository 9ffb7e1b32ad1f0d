mkdir -p gpurun_out
PYTHONPATH=. timeout 200 python tools/dbg_stream.py b 4 40 > gpurun_out/dbg18.log 2>&1; echo dbg=$?
grep -v "wait timeout" gpurun_out/dbg18.log | tail -4; grep -c "wait timeout" gpurun_out/dbg18.log; grep "wait timeout" gpurun_out/dbg18.log | head -3
