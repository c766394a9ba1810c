#!/bin/bash
# round 2, pass 7: A/B of PAIR4 with two parameter copies of column 0, and of a
# two-step Montgomery-64 loop body
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/pair2.so $L/_lib_var/pair4c.so $L/_lib_var/pair2.so $L/_lib_var/pair4c.so; do
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 1 10 >> gpurun_out/r2c7_ab_pair4c.txt 2>&1
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 0 10 >> gpurun_out/r2c7_ab_pair4c.txt 2>&1
done
for lib in $L/_lib_var/wideu1.so $L/_lib_var/wideu2.so $L/_lib_var/widealu.so $L/_lib_var/wideu1.so $L/_lib_var/wideu2.so $L/_lib_var/widealu.so; do
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 35 36 --bits 32 --only wide1 --out gpurun_out/r2c7_$(basename $lib .so).json >> gpurun_out/r2c7_wide_unroll.log 2>&1
done
for lib in $L/_lib_var/alu0.so $L/_lib_var/alu1.so $L/_lib_var/alu0.so $L/_lib_var/alu1.so; do
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 35 36 --bits 34 --only red3 red1 lazy3 --out gpurun_out/r2c7_$(basename $lib .so).json >> gpurun_out/r2c7_alu_add.log 2>&1
done
