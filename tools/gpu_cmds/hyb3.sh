timeout 600 python -m pytest tests -m gpu -q -x -k "hybrid" > gpurun_out/gpu_hyb3.log 2>&1; tail -2 gpurun_out/gpu_hyb3.log
timeout 900 python tools/modp_rates.py 24 28 32 36 40 --only hyb11 --out gpurun_out/modp_rates_hyb3.json > gpurun_out/modp_rates_hyb3.log 2>&1; cut -c1-300 gpurun_out/modp_rates_hyb3.log
