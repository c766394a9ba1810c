#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/wp1.so $L/_lib_var/wp2.so $L/_lib_var/wp2u1.so $L/_lib_var/wp1.so $L/_lib_var/wp2.so $L/_lib_var/wp2u1.so; do
  echo "== $lib" >> gpurun_out/r2c17_wide.log
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 32 35 36 --bits 34 --only wide2 --out /tmp/x.json >> gpurun_out/r2c17_wide.log 2>&1
done
