# Montgomery-64 column-sum REDC: mul.hi + adds (PK_REDC64_PS=1) vs madc.hi.cc (=2)
mkdir -p gpurun_out
for n in 35 36; do
  for L in paper_2602_10141_b200/_lib_var/ps1.so paper_2602_10141_b200/_lib_var/ps2.so paper_2602_10141_b200/_lib_var/ps1.so paper_2602_10141_b200/_lib_var/ps2.so; do
    PERMKIT_GPU_LIB=$L timeout 300 python tools/redc_ab.py $n 34
  done
done > gpurun_out/redc_ps2.log 2>&1
cut -c1-250 gpurun_out/redc_ps2.log
