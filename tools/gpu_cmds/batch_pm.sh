# A/B: batched kernel (per-warp matrix slots) vs one C0P launch per matrix over 4 streams
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv | tee gpurun_out/batch_pm_smi.log
nproc
for n in 20 22 23 24 26 28; do for f in 0 1; do PK_BATCH_PER_MATRIX=$f python tools/prof_one.py batch $n 2048 3 | sed "s/^/pm=$f /"; done; done 2>&1 | tee gpurun_out/batch_pm.log
for f in 0 1; do PK_BATCH_PER_MATRIX=$f python tools/prof_one.py batchr 26 1024 2 | sed "s/^/pm=$f /"; done 2>&1 | tee -a gpurun_out/batch_pm.log
timeout 1200 python -m pytest tests -m gpu -q -x -k "batch or sample or c5 or c1 or geodesic or ensemble" > gpurun_out/gpu_pm.log 2>&1; tail -3 gpurun_out/gpu_pm.log
timeout 900 python bench.py > gpurun_out/bench_pm.json 2> gpurun_out/bench_pm.err; tail -c 700 gpurun_out/bench_pm.json
