# round deliverables after the latency work: default bench line, reference arm,
# GPU tests, ncu launch list + full capture of the stream kernel and the batched update
mkdir -p gpurun_out /tmp/rep
TAG=${1:-r01p}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.jsonl 2> gpurun_out/${TAG}_bench_ref.err; echo ref=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-queries --twopass-n 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_streams --launch-skip 2 -c 1 -o /tmp/rep/${TAG}_stream $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full=$?
ncu -i /tmp/rep/${TAG}_stream.ncu-rep --page raw --csv > gpurun_out/${TAG}_stream_raw.csv 2>/dev/null
ncu -i /tmp/rep/${TAG}_stream.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_stream_src.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_word_logprob_ring -c 1 -o /tmp/rep/${TAG}_hsq python tools/qbench.py tf32x3 1 > gpurun_out/${TAG}_ncu_hsq.log 2>&1; echo hsq=$?
ncu -i /tmp/rep/${TAG}_hsq.ncu-rep --page raw --csv > gpurun_out/${TAG}_hsq_raw.csv 2>/dev/null
ls -la gpurun_out | tail -20
