timeout 900 python -m pytest tests -m gpu -q -x -k "hybrid or resident" > gpurun_out/gpu_hybdadd.log 2>&1; tail -2 gpurun_out/gpu_hybdadd.log
timeout 900 python tools/modp_rates.py 24 32 36 40 --only hyb11 hybw11 --out gpurun_out/modp_rates_hybdadd.json 2>&1 | cut -c1-250
