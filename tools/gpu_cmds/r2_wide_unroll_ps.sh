# Montgomery-64 steps per loop body (PK_WIDE_UNROLL 1 / 2 / 3) with the form-2 REDC
mkdir -p gpurun_out
for n in 35 36; do
  for u in 1 2 3 2; do
    PERMKIT_GPU_LIB=paper_2602_10141_b200/_lib_var/u$u.so timeout 300 python tools/redc_ab.py $n 34
  done
done > gpurun_out/wide_unroll_ps.log 2>&1
cut -c1-250 gpurun_out/wide_unroll_ps.log
