timeout 900 python -m pytest tests -m gpu -q -x -k "hybrid or schur or resident or wide or modp" > gpurun_out/gpu_hybw.log 2>&1; tail -3 gpurun_out/gpu_hybw.log
timeout 900 python tools/modp_rates.py 24 32 36 40 --only hyb11 hybw11 red3 --out gpurun_out/modp_rates_hybw.json > gpurun_out/modp_rates_hybw.log 2>&1; cut -c1-300 gpurun_out/modp_rates_hybw.log
