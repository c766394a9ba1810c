timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_c0p.log 2>&1; tail -3 gpurun_out/gpu_c0p.log
timeout 900 python bench.py > gpurun_out/bench_c0p.json 2> gpurun_out/bench_c0p.err; tail -c 3000 gpurun_out/bench_c0p.json
