timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all2.log 2>&1; tail -3 gpurun_out/gpu_all2.log
timeout 600 python -c "
import time
from paper_2602_10141_b200 import modular
modular.schur_permanent_exact(21)
for n in (33, 35, 36):
    t=time.perf_counter(); v,b,w=modular.schur_permanent_exact(n); dt=time.perf_counter()-t
    print(n, v, len(b.primes), 'primes, default 59-bit basis', round(dt,3), 's', flush=True)
" 2>&1 | tee gpurun_out/schur59b.log
timeout 1800 python tools/schur_run.py 39 41 43 --out gpurun_out/schur_c4b.json > gpurun_out/schur_c4b.log 2>&1; cut -c1-400 gpurun_out/schur_c4b.log
