# ncu --set full of the Montgomery-64 walk with the column-sum REDC (form 2), n = 36
mkdir -p gpurun_out
timeout 300 python tools/prof_one.py wide 36 1 30 > gpurun_out/r2_wide_ps_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -c 1 -k regex:walk_modp64 -o gpurun_out/r2_wide36_ps python tools/prof_one.py wide 36 1 30 > gpurun_out/r2_wide_ps_ncu.log 2>&1
tail -2 gpurun_out/r2_wide_ps_ncu.log
