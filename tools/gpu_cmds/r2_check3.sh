#!/bin/bash
# round 2, pass 3: plan-level perm_blocked (parity + timing), col0 layout A/B,
# ncu captures of the F_p launch groups behind the bench's CRT rooflines
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
L=paper_2602_10141_b200
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "plan or blocked or multidev or unaligned or production or tile or split" > gpurun_out/r2c3_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c3_pytest.txt
for nb in "24 512" "28 512" "20 64"; do timeout 120 python tools/plan_timing.py $nb >> gpurun_out/r2c3_plan_timing.txt 2>&1; done
for lib in $L/_lib_var/r1.so $L/_lib_var/col0a.so $L/_lib_var/col0s.so $L/_lib_var/r1.so $L/_lib_var/col0a.so $L/_lib_var/col0s.so; do
  PERMKIT_GPU_LIB=$lib timeout 120 python tools/ab_f64.py 32 1 10 >> gpurun_out/r2c3_ab_f64.txt 2>&1
done
NCU="ncu --set full --import-source on --clock-control none -c 1"
timeout 600 $NCU -k regex:walk_modp64 -o gpurun_out/r2_wide36 python tools/prof_one.py wide 36 1 30 > gpurun_out/r2c3_ncu_wide.log 2>&1
timeout 600 $NCU -k regex:walk_hybrid -o gpurun_out/r2_hybw36 python tools/prof_one.py basis 36 1 32 > gpurun_out/r2c3_ncu_hybw.log 2>&1
timeout 600 $NCU -k regex:walk_modp_kernel -o gpurun_out/r2_red3_35 python tools/prof_one.py red3 35 1 32 > gpurun_out/r2c3_ncu_red3.log 2>&1
