timeout 1500 python -m pytest tests -m gpu -q -x -k "schur or hybrid or wide or modp or resident" > gpurun_out/gpu_glynn.log 2>&1; tail -3 gpurun_out/gpu_glynn.log
timeout 2400 python tools/schur_run.py 35 36 37 39 41 43 --check 37 --out gpurun_out/schur_glynn.json > gpurun_out/schur_glynn.log 2>&1; cut -c1-300 gpurun_out/schur_glynn.log
