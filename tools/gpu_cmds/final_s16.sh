# final round-1 validation after the 16-stream / m >= 20 (complex), m >= 21 (real) switch
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_fin16.log 2>&1; tail -3 gpurun_out/gpu_fin16.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_fin16.log 2>&1; tail -1 gpurun_out/smoke_fin16.log
timeout 900 python bench.py > gpurun_out/bench_fin16.json 2> gpurun_out/bench_fin16.err; tail -c 400 gpurun_out/bench_fin16.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fin16.csv python bench.py --steps 2 --warmup 3 --no-secondary > gpurun_out/ncu_launch_fin16.log 2>&1; tail -1 gpurun_out/ncu_launch_fin16.log
timeout 1200 python tools/configs_run.py > gpurun_out/configs_fin16.jsonl 2>&1; cat gpurun_out/configs_fin16.jsonl | cut -c1-200
