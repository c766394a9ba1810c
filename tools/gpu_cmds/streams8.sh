# per-matrix batched launches over 8 streams from m = 21; full GPU suite, smoke, bench, launch list
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv > gpurun_out/s8_smi.log
for n in 20 21; do for f in 0 1; do PK_BATCH_PER_MATRIX=$f python tools/prof_one.py batch $n 2048 3 | sed "s/^/pm=$f /"; done; done > gpurun_out/s8_batch.log 2>&1
for n in 22 23 24 26; do python tools/prof_one.py batch $n 2048 2; done >> gpurun_out/s8_batch.log 2>&1; cat gpurun_out/s8_batch.log | cut -c1-200
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_s8.log 2>&1; tail -3 gpurun_out/gpu_s8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s8.log 2>&1; tail -1 gpurun_out/smoke_s8.log
timeout 900 python bench.py > gpurun_out/bench_s8.json 2> gpurun_out/bench_s8.err; tail -c 1500 gpurun_out/bench_s8.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s8.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_s8.log 2>&1; tail -2 gpurun_out/ncu_launch_s8.log
