mkdir -p gpurun_out
for a in "tf32x3 16 stream" "tf32x3 16 level" "fp64 16 level"; do
  set -- $a
  PYTHONPATH=. timeout 600 python tools/tie_check.py $1 $2 $3 > gpurun_out/tie_$1_$3.json 2> gpurun_out/tie_$1_$3.err; echo $1 $3 rc=$?
done
