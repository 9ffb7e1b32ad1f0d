# round-end check of HEAD: GPU tests, default bench line, bench under torchrun (NCCL, world 1), reference arm under torchrun
mkdir -p gpurun_out
TAG=${1:-r01j}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-queries --twopass-n 0 > gpurun_out/${TAG}_bench_torchrun.jsonl 2> gpurun_out/${TAG}_bench_torchrun.err; echo torchrun=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref_torchrun.jsonl 2> gpurun_out/${TAG}_bench_ref_torchrun.err; echo ref_torchrun=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$?
