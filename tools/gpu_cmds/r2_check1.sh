#!/bin/bash
# round 2, first GPU pass: full GPU suite + bench (both arms) + SASS-vs-ncu for the CRT groups
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2c1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c1_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c1_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c1_bench.json 2> gpurun_out/r2c1_bench.err
echo "bench rc=$?" >> gpurun_out/r2c1_bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2c1_ref.json 2> gpurun_out/r2c1_ref.err
echo "ref rc=$?" >> gpurun_out/r2c1_ref.err
