cd tools/micro && for b in walk_ccol0 walk_ccol1 walk_ccol0_nk walk_r_ccol0 walk_r_ccol1; do timeout 60 ./$b; done 2>&1 | tee ../../gpurun_out/walk_exp4.log
