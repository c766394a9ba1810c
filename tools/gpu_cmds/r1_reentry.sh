timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_re.log 2>&1; tail -3 gpurun_out/gpu_re.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_re.log 2>&1; tail -1 gpurun_out/smoke_re.log
timeout 900 python bench.py > gpurun_out/bench_re.json 2> gpurun_out/bench_re.err; tail -c 600 gpurun_out/bench_re.json
for n in 20 23 24 26 28; do python tools/prof_one.py batch $n 2048; done > gpurun_out/batch_re.log 2>&1; cat gpurun_out/batch_re.log | cut -c1-300
