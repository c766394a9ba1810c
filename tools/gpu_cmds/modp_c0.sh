timeout 900 python -m pytest tests -m gpu -q -x -k "modp or schur or hybrid or wide or exact_integers or engine" > gpurun_out/gpu_modpc0.log 2>&1; tail -3 gpurun_out/gpu_modpc0.log
timeout 900 python tools/modp_rates.py 32 36 40 --out gpurun_out/modp_rates_c0.json > gpurun_out/modp_rates_c0.log 2>&1; cut -c1-400 gpurun_out/modp_rates_c0.log
