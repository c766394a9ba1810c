#!/bin/bash
# complex fp64 walk rate at n = 42..46 over 2^13 tiles each (k = n - 22, range = 2^(k+5+13)):
# the register-spilling sizes 44/46 vs 43/45
mkdir -p gpurun_out
for n in 42 43 44 45 46; do
  timeout 300 python tools/prof_one.py f64c $n 1 $((n - 22 + 18))
done > gpurun_out/r2_f64c_large.txt 2>&1
echo rc=$?
