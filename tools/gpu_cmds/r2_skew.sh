#!/bin/bash
# block kernel: 4 steps in flight (product) vs 8 real / 6 complex
mkdir -p gpurun_out
for v in skew4 skew8r; do
  PERMKIT_GPU_LIB=paper_2602_10141_b200/_lib_var/$v.so timeout 600 python tools/block_rate.py > gpurun_out/r2k_$v.jsonl 2>&1
  echo "$v rc=$?"
done
