# per-matrix batched launches: 8 / 12 / 16 streams at n = 20-26 (m = 20 launches are 32 CTAs)
{
PK_BATCH_PER_MATRIX=0 python tools/prof_one.py batch 20 2048 3 | sed "s/^/pm=0 /"
for n in 20 21; do for st in 8 12 16; do PK_BATCH_PER_MATRIX=1 PK_BATCH_STREAMS=$st python tools/prof_one.py batch $n 2048 3 | sed "s/^/pm=1 st=$st /"; done; done
for n in 19; do PK_BATCH_PER_MATRIX=0 python tools/prof_one.py batch $n 2048 3 | sed "s/^/pm=0 /"; PK_BATCH_PER_MATRIX=1 PK_BATCH_STREAMS=16 python tools/prof_one.py batch $n 2048 3 | sed "s/^/pm=1 st=16 /"; done
for n in 23 26; do for st in 8 16; do PK_BATCH_PER_MATRIX=1 PK_BATCH_STREAMS=$st python tools/prof_one.py batch $n 2048 2 | sed "s/^/pm=1 st=$st /"; done; done
} > gpurun_out/s16_batch.log 2>&1; cat gpurun_out/s16_batch.log
