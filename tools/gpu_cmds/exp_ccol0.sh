cd tools/micro && for b in walk_base walk_ccol0 walk_cw walk_ccol0_t2u2 walk_r_base walk_r_ccol0; do timeout 60 ./$b; done > ../../gpurun_out/walk_exp3.log 2>&1; cd ../..; cat gpurun_out/walk_exp3.log
timeout 900 python -m pytest tests -m gpu -q -x -k "schur or hybrid or wide" > gpurun_out/gpu_basis.log 2>&1; tail -3 gpurun_out/gpu_basis.log
