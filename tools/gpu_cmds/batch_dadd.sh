for n in 20 23 24 26 28; do python tools/prof_one.py batch $n 2048; done
python tools/prof_one.py f64c 44 1 40; python tools/prof_one.py f64c 48 1 42
timeout 2400 python -m pytest tests -m gpu -q -x -k "f64 or tile or full or exact or unaligned or device_split or batch or large_n or c1 or c5 or geodesic or engine or blocked or resident or glynn_naive or production" > gpurun_out/gpu_bdadd.log 2>&1; tail -3 gpurun_out/gpu_bdadd.log
