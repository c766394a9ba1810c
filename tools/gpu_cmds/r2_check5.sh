#!/bin/bash
# round 2, pass 5: real fp64 walks to n = 64 (parity + 54 x 54 extrapolation),
# the complex mix ceiling in the bench, 4-term Neumaier A/B
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
timeout 900 python -m pytest tests/test_gpu_real64.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "real or large_n or limits or full_permanent" > gpurun_out/r2c5_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c5_pytest.txt
timeout 600 python tools/real54_rate.py 49 54 60 64 > gpurun_out/r2c5_real54.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c5_bench.json 2> gpurun_out/r2c5_bench.err
for lib in $L/_lib_var/pair2.so $L/_lib_var/pair4.so $L/_lib_var/pair2.so $L/_lib_var/pair4.so; do
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 1 10 >> gpurun_out/r2c5_ab_pair4.txt 2>&1
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 0 10 >> gpurun_out/r2c5_ab_pair4.txt 2>&1
done
