timeout 900 python -m pytest tests -m gpu -q -x -k "wide or schur_default" > gpurun_out/gpu_wide2.log 2>&1; tail -3 gpurun_out/gpu_wide2.log
timeout 900 python tools/modp_rates.py 20 32 36 40 --only wide1 wide2 --out gpurun_out/modp_rates_wide2.json > gpurun_out/modp_rates_wide2.log 2>&1; cut -c1-300 gpurun_out/modp_rates_wide2.log
