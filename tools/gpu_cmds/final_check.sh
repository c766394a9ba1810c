# final round-1 check of the committed build: GPU tests and smoke
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_final.log 2>&1; tail -2 gpurun_out/gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -1 gpurun_out/smoke_final.log
