#!/bin/bash
# round 2, pass 10: full GPU suite (signed-integer max-size gate, PAIR4 off) + bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c10_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c10_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c10_bench.json 2> gpurun_out/r2c10_bench.err
