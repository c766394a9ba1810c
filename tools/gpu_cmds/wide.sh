set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "wide or schur_default or modp or schur_exact" > gpurun_out/gpu_wide.log 2>&1; tail -5 gpurun_out/gpu_wide.log
timeout 600 python tools/modp_rates.py 20 32 36 43 --only wide1 wide2 --out gpurun_out/modp_rates_wide.json > gpurun_out/modp_rates_wide.log 2>&1; cat gpurun_out/modp_rates_wide.log
timeout 600 python -c "
import time
from paper_2602_10141_b200 import modular
modular.schur_permanent_exact(21)
for n in (31, 33, 35, 36):
    t=time.perf_counter(); v,b,w=modular.schur_permanent_exact(n); dt=time.perf_counter()-t
    print(n, v, [len(b.primes)], 'default 59-bit basis', round(dt,3), 's', flush=True)
" 2>&1 | tee gpurun_out/schur59.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all.log 2>&1; tail -3 gpurun_out/gpu_all.log
