cd tools/micro && for b in walk_final walk_r_final; do timeout 60 ./$b; done 2>&1 | tee ../../gpurun_out/walk_exp8.log; cd ../..
timeout 2400 python -m pytest tests -m gpu -q -x -k "f64 or tile or full or exact or unaligned or device_split or batch or large_n or c1 or c5 or geodesic or engine or blocked or resident or glynn_naive or production" > gpurun_out/gpu_dadd.log 2>&1; tail -3 gpurun_out/gpu_dadd.log
timeout 900 python bench.py --no-secondary > gpurun_out/bench_dadd.json 2>/dev/null; tail -c 600 gpurun_out/bench_dadd.json
