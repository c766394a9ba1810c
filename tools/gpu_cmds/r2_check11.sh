#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_real64.py tests/test_gpu_multidev.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/r2c11_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c11_pytest.txt
