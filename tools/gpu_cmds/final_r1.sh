timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_final.log 2>&1; tail -3 gpurun_out/gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -2 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 2500 gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-secondary > gpurun_out/ncu_launch_final.log 2>&1
timeout 600 python -c "
import time
from paper_2602_10141_b200 import modular
modular.schur_permanent_exact(21)
for n in (33, 35, 36):
    t=time.perf_counter(); v,b,w=modular.schur_permanent_exact(n); dt=time.perf_counter()-t
    print(n, v, len(b.primes), 'primes, default 59-bit basis, glynn', round(dt,3), 's', flush=True)
" 2>&1 | tee gpurun_out/schur59_final.log
