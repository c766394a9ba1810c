timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_hybw2.log 2>&1; tail -3 gpurun_out/gpu_hybw2.log
timeout 1200 python tools/schur_run.py 35 36 39 41 --check 36 --out gpurun_out/schur_hybw.json > gpurun_out/schur_hybw.log 2>&1; cut -c1-330 gpurun_out/schur_hybw.log
