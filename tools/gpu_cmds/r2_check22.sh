#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/wc0.so $L/_lib_var/wca.so $L/_lib_var/wcu1.so $L/_lib_var/wc0.so $L/_lib_var/wca.so $L/_lib_var/wcu1.so; do
  echo "== $lib" >> gpurun_out/r2c22_wide.log
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 32 35 36 --bits 34 --only wide1 --out /tmp/x.json >> gpurun_out/r2c22_wide.log 2>&1
done
