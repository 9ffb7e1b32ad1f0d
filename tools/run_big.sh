set -u
timeout 900 python tools/sched_e.py > gpurun_out/sched_e.jsonl 2> gpurun_out/sched_e.err
OTFLM_HS_TC=0 timeout 900 python tools/sched_e.py > gpurun_out/sched_e_f64.jsonl 2>> gpurun_out/sched_e.err
