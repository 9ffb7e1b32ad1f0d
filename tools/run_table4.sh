python -c "
import sys, json; sys.path.insert(0,'.')
import bench
print(json.dumps(bench.table4_sweep('exact')))
" > gpurun_out/r02ad_table4.json 2> gpurun_out/r02ad_table4.err
tail -3 gpurun_out/r02ad_table4.err
