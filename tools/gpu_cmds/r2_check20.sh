#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
for lib in $L/_lib_var/wcb.so $L/_lib_var/wci.so $L/_lib_var/wcb.so $L/_lib_var/wci.so; do
  echo "== $lib" >> gpurun_out/r2c20_wide.log
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 32 35 36 --bits 34 --only wide1 --out /tmp/x.json >> gpurun_out/r2c20_wide.log 2>&1
  PERMKIT_GPU_LIB=$lib timeout 300 python -c "
from paper_2602_10141_b200 import modular
v=-15139017417029296875
for p in modular.find_primes(35).primes:
    r=modular.schur_residue(35, p).residue
    print('check', p, r == v % p)
" >> gpurun_out/r2c20_wide.log 2>&1
done
