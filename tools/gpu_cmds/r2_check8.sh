#!/bin/bash
# round 2, pass 8: Montgomery-64 two-step body / ALU-add A/B, Montgomery-32 ALU-add A/B
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/wideu1.so $L/_lib_var/wideu2.so $L/_lib_var/widealu.so $L/_lib_var/wideu1.so $L/_lib_var/wideu2.so $L/_lib_var/widealu.so; do
  echo "== $lib" >> gpurun_out/r2c8_wide.log
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 35 36 --bits 32 --only wide1 --out /tmp/x.json >> gpurun_out/r2c8_wide.log 2>&1
done
for lib in $L/_lib_var/alu0.so $L/_lib_var/alu1.so $L/_lib_var/alu0.so $L/_lib_var/alu1.so; do
  echo "== $lib" >> gpurun_out/r2c8_alu.log
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 35 36 --bits 34 --only red3 red1 lazy3 --out /tmp/x.json >> gpurun_out/r2c8_alu.log 2>&1
done
