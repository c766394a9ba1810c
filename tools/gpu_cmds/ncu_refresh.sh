# refresh the full ncu captures of the headline walks with the committed code
python tools/prof_one.py f64c 32 > gpurun_out/pre_f64c.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_f64 -c 1 -f -o gpurun_out/prof_f64c32_fin python tools/prof_one.py f64c 32 > gpurun_out/ncu_f64c_fin.log 2>&1; tail -1 gpurun_out/ncu_f64c_fin.log
python tools/prof_one.py f64r 32 > gpurun_out/pre_f64r.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_f64 -c 1 -f -o gpurun_out/prof_f64r32_fin python tools/prof_one.py f64r 32 > gpurun_out/ncu_f64r_fin.log 2>&1; tail -1 gpurun_out/ncu_f64r_fin.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_f64 -s 8 -c 1 -f -o gpurun_out/prof_batch21_fin python tools/prof_one.py batch 21 256 > gpurun_out/ncu_b21_fin.log 2>&1; tail -1 gpurun_out/ncu_b21_fin.log
