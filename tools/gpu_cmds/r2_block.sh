#!/bin/bash
# A/B of the exact per-block kernel: round-2 library (old local-memory state) vs the
# register-state NMAX templates with skewed passes; then the block parity tests.
mkdir -p gpurun_out
for v in oldblock newblock; do
  PERMKIT_GPU_LIB=paper_2602_10141_b200/_lib_var/$v.so timeout 600 python tools/block_rate.py > gpurun_out/r2b_$v.jsonl 2>&1
  echo "$v rc=$?"
done
timeout 1200 python -m pytest tests -m gpu -x -q -k "block or plan or blocked or ragged or exact or modp or batch" > gpurun_out/r2b_pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2b_pytest.txt
