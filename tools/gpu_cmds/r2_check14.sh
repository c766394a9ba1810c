#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/wu2.so $L/_lib_var/wu3.so $L/_lib_var/wu4.so $L/_lib_var/wu2.so $L/_lib_var/wu3.so $L/_lib_var/wu4.so; do
  echo "== $lib" >> gpurun_out/r2c14_wide.log
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 32 36 --bits 34 --only wide1 --out /tmp/x.json >> gpurun_out/r2c14_wide.log 2>&1
done
