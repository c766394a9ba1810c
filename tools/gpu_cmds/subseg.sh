cd tools/micro && for b in walk_sub walk_r_sub; do timeout 60 ./$b; done 2>&1 | tee ../../gpurun_out/walk_exp6.log; cd ../..
python tools/prof_one.py f64c 36 1; python tools/prof_one.py f64c 40 1 34; python tools/prof_one.py f64r 40 1 36
timeout 2400 python -m pytest tests -m gpu -q -x -k "f64 or tile or full or exact or unaligned or device_split or batch or large_n or c1 or c5 or geodesic or engine or blocked or resident or glynn_naive" > gpurun_out/gpu_subseg.log 2>&1; tail -3 gpurun_out/gpu_subseg.log
