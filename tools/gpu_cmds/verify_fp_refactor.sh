set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests2.log 2>&1; tail -3 gpurun_out/gpu_tests2.log
cd tools/micro && for b in walk_base walk_tree2 walk_unr2 walk_tree2_unr2 walk_r_base walk_r_tree2 walk_r_unr2; do timeout 60 ./$b; done > ../../gpurun_out/walk_exp2.log 2>&1; cd ../..; cat gpurun_out/walk_exp2.log
timeout 900 python tools/modp_rates.py 32 36 40 43 > gpurun_out/modp_rates.log 2>&1; tail -30 gpurun_out/modp_rates.log
