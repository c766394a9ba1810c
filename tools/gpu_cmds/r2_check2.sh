#!/bin/bash
# round 2, pass 2: parity of the rewritten F_p kernels, hybrid / wide A/B, the
# hybrid mix ceiling, and the headline walk against the round-1 library
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "wide or hybrid or schur or modp or multidev or resident" > gpurun_out/r2c2_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c2_pytest.txt
L=paper_2602_10141_b200
timeout 300 python tools/modp_rates.py 35 36 --bits 34 --only hybw11 hyb11 wide1 red3 red1 --out gpurun_out/r2c2_rates_main.json > gpurun_out/r2c2_rates_main.log 2>&1
for lib in $L/_lib_var/hybtree0.so $L/_lib_var/hybt1m3.so $L/_lib_var/hybt0m3.so $L/_lib_var/hybtree1.so; do
  tag=$(basename $lib .so)
  PERMKIT_GPU_LIB=$lib timeout 300 python tools/modp_rates.py 35 36 --bits 34 --only hybw11 hyb11 --out gpurun_out/r2c2_rates_$tag.json > gpurun_out/r2c2_rates_$tag.log 2>&1
done
timeout 300 tools/micro/hybrid_mix > gpurun_out/r2c2_hybrid_mix.txt 2>&1
for lib in $L/_lib_var/r1.so $L/_lib/libpermkit_gpu.so $L/_lib_var/r1.so $L/_lib/libpermkit_gpu.so; do
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 1 10 >> gpurun_out/r2c2_ab_f64.txt 2>&1
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 0 10 >> gpurun_out/r2c2_ab_f64.txt 2>&1
done
