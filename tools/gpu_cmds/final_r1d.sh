timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_final4.log 2>&1; tail -3 gpurun_out/gpu_final4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final4.log 2>&1; tail -1 gpurun_out/smoke_final4.log
timeout 900 python bench.py > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err; tail -c 900 gpurun_out/bench_final4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final4.csv python bench.py --steps 2 --warmup 1 --no-secondary > gpurun_out/ncu_launch_final4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_f64 -s 8 -c 1 -f -o gpurun_out/prof_batch_pm23 python tools/prof_one.py batch 23 256 > gpurun_out/ncu_batch_pm23.log 2>&1; tail -1 gpurun_out/ncu_batch_pm23.log
