# A/B of library variants in var_so/: default bench line (phase timers) + config-c phases each
mkdir -p gpurun_out
TAG=${1:-ab}
cp paper_2007_11794_b200/libotflm_b200.so /tmp/lib_main.so
for v in var_so/lib_*.so; do
  n=$(basename $v .so)
  cp $v paper_2007_11794_b200/libotflm_b200.so
  timeout 300 python bench.py --no-cpu-baseline --no-queries --twopass-n 0 > gpurun_out/${TAG}_${n}_bench.jsonl 2> gpurun_out/${TAG}_${n}_bench.err; echo $n bench=$?
  timeout 300 python tools/phases_c.py > gpurun_out/${TAG}_${n}_phc.json 2> gpurun_out/${TAG}_${n}_phc.err; echo $n phc=$?
done
cp /tmp/lib_main.so paper_2007_11794_b200/libotflm_b200.so
