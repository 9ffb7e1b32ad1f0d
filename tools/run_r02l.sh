python bench.py --e-total 296 --steps 2 --warmup 1 --out gpurun_out/r02l_small.json > gpurun_out/r02l_small.log 2>&1
echo "small rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 --out gpurun_out/r02l_ref.json > gpurun_out/r02l_ref.log 2>&1
echo "ref rc=$?"
/usr/bin/time -v python bench.py --out gpurun_out/r02l_full.json > gpurun_out/r02l_full.log 2>&1
echo "full rc=$?"
tail -n 5 gpurun_out/r02l_small.log | cut -c1-400
