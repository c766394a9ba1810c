# Montgomery-64 product-scanning REDC (PK_REDC64_PS) A/B: identical residues and rates
mkdir -p gpurun_out
for n in 32 35 36; do
  for L in product paper_2602_10141_b200/_lib_var/ps0.so paper_2602_10141_b200/_lib_var/ps1.so; do
    if [ $L = product ]; then unset PERMKIT_GPU_LIB; else export PERMKIT_GPU_LIB=$L; fi
    timeout 300 python tools/redc_ab.py $n 34
  done
done > gpurun_out/redc_ps.log 2>&1
for L in paper_2602_10141_b200/_lib_var/ps0.so paper_2602_10141_b200/_lib_var/ps1.so; do
  PERMKIT_GPU_LIB=$L timeout 300 python tools/redc_ab.py 36 34
done >> gpurun_out/redc_ps.log 2>&1
cat gpurun_out/redc_ps.log | cut -c1-400
