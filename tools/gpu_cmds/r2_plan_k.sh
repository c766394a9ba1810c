# Segment-size (k) sweep of the fp64 headline walk and the F_p n = 36 groups (PK_PLAN_K hook)
mkdir -p gpurun_out
L=paper_2602_10141_b200/_lib/libpermkit_gpu.so
for K in 0 9 10 11 12 13 14; do
  if [ $K = 0 ]; then unset PK_PLAN_K; else export PK_PLAN_K=$K; fi
  echo "K=$K $(PERMKIT_GPU_LIB=$L timeout 300 python tools/ab_f64.py 32 1 10)"
done > gpurun_out/plan_k_f64.log 2>&1
unset PK_PLAN_K
for K in 0 12 13 15 16; do
  if [ $K = 0 ]; then unset PK_PLAN_K; else export PK_PLAN_K=$K; fi
  echo "K=$K"; timeout 600 python tools/modp_rates.py 36 --bits 35 --only hybw11 red3 --out gpurun_out/plan_k_modp_$K.json 2>&1 | cut -c1-200
done > gpurun_out/plan_k_modp.log 2>&1
cat gpurun_out/plan_k_f64.log; cat gpurun_out/plan_k_modp.log
