#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/mu1.so $L/_lib_var/mu2.so $L/_lib_var/mu1.so $L/_lib_var/mu2.so; do
  echo "== $lib" >> gpurun_out/r2c15_modp.log
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 35 36 --bits 34 --only red3 red1 lazy3 hyb11 hybw11 --out /tmp/x.json >> gpurun_out/r2c15_modp.log 2>&1
done
