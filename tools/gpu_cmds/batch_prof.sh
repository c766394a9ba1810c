python tools/prof_one.py f64c 23 20
python tools/prof_one.py f64c 24 20
python tools/prof_one.py batch 23 4096
python tools/prof_one.py batch 24 4096
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_f64 -c 1 -f -o gpurun_out/prof_batch23 python tools/prof_one.py batch 23 4096 > gpurun_out/ncu_batch23.log 2>&1; tail -2 gpurun_out/ncu_batch23.log
