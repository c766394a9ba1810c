#!/bin/bash
# CIOS Montgomery-64 in the main build: every F_p / wide parity test, the bench, ncu of the wide walk
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "modp or wide or schur or multidev or exact or integers or kats or resident" > gpurun_out/r2c21_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c21_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c21_bench.json 2> gpurun_out/r2c21_bench.err
timeout 900 python tools/modp_rates.py 32 35 36 --bits 34 --only wide1 red3 hybw11 > gpurun_out/r2c21_rates.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -c 1 -k regex:walk_modp64 -o gpurun_out/r2_wide36c python tools/prof_one.py wide 36 1 30 > gpurun_out/r2c21_ncu.log 2>&1
