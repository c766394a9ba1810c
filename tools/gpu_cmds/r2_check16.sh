#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/bs0.so $L/_lib_var/bs1.so $L/_lib_var/bs0.so $L/_lib_var/bs1.so $L/_lib_var/bs0.so $L/_lib_var/bs1.so; do
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 1 10 >> gpurun_out/r2c16_ab_blocksum.txt 2>&1
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 0 10 >> gpurun_out/r2c16_ab_blocksum.txt 2>&1
done
