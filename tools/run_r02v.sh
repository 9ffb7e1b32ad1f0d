python tools/decode_once.py e 74 300 exact > gpurun_out/r02v_plain.log 2>&1 && \
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-queries > gpurun_out/r02v_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02v_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-queries > gpurun_out/r02v_launches_run.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_decode_streams -c 1 -o gpurun_out/r02v_stream_e python tools/decode_once.py e 74 300 exact > gpurun_out/r02v_ncu.log 2>&1
echo done
