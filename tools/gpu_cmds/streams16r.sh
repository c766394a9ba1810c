# real (float64) batches: per-matrix (16 streams) vs per-warp-slot at m = 20-23
for n in 20 21 22 23; do for f in 0 1; do PK_BATCH_PER_MATRIX=$f python tools/prof_one.py batchr $n 2048 3 | sed "s/^/pm=$f /"; done; done > gpurun_out/s16r_batch.log 2>&1; cat gpurun_out/s16r_batch.log
python tools/prof_one.py batchr 22 2048 2; python tools/prof_one.py batch 20 2048 2
