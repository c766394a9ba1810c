# per-matrix batched launches: stream count and the m threshold
for n in 21 22 23 24; do
  PK_BATCH_PER_MATRIX=0 python tools/prof_one.py batch $n 2048 3 | sed "s/^/pm=0 /"
  for st in 2 4 8; do PK_BATCH_PER_MATRIX=1 PK_BATCH_STREAMS=$st python tools/prof_one.py batch $n 2048 3 | sed "s/^/pm=1 st=$st /"; done
done 2>&1 | tee gpurun_out/batch_streams.log
