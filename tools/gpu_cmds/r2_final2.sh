#!/bin/bash
# round 2, final pass 2: the reference-pinned perm(S_35 / 37) tests and the bench with the n = 37 golden
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "schur or integration" > gpurun_out/r2f2_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f2_pytest.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f2_bench.json 2> gpurun_out/r2f2_bench.err
