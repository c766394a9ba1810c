# adopted: 16 streams, per-matrix from m = 20; batch tests, A/B lines, bench
{ for n in 20 21 22 23; do python tools/prof_one.py batch $n 2048 3; done; PK_BATCH_PER_MATRIX=0 python tools/prof_one.py batch 20 2048 3 | sed "s/^/pm=0 /"; python tools/prof_one.py batchr 20 2048 3; PK_BATCH_PER_MATRIX=0 python tools/prof_one.py batchr 20 2048 3 | sed "s/^/pm=0 /"; } > gpurun_out/s16b_batch.log 2>&1; cat gpurun_out/s16b_batch.log
timeout 1200 python -m pytest tests -m gpu -q -x -k "batch or sample or c5 or c1 or geodesic or ensemble or sweep" > gpurun_out/gpu_s16.log 2>&1; tail -3 gpurun_out/gpu_s16.log
timeout 900 python bench.py > gpurun_out/bench_s16.json 2> gpurun_out/bench_s16.err; tail -c 400 gpurun_out/bench_s16.json
