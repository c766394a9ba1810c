timeout 1800 python -m pytest tests -m gpu -q -x -k "large_n" --durations=10 > gpurun_out/gpu_large.log 2>&1; tail -20 gpurun_out/gpu_large.log
