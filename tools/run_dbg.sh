mkdir -p gpurun_out
PYTHONPATH=. timeout 100 python tools/dbg_stream.py a 12 60 > gpurun_out/dbg5.log 2>&1; echo dbg5=$?
grep -v "^hs ring" gpurun_out/dbg5.log | head -20
PYTHONPATH=. timeout 400 compute-sanitizer --tool memcheck --print-limit 10 python tools/dbg_stream.py b 2 10 > gpurun_out/dbg4.log 2>&1; echo dbg4=$?
grep -v "^=========     " gpurun_out/dbg4.log | head -50
