#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multidev.py -m gpu -q -p no:cacheprovider -k "concurrent or plan" > gpurun_out/r2c18_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c18_pytest.txt
PK_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 8 --steps 2 --warmup 1 > gpurun_out/r2c18_bench_n8.json 2> gpurun_out/r2c18_bench_n8.err
echo "n8 rc=$?" >> gpurun_out/r2c18_bench_n8.err
