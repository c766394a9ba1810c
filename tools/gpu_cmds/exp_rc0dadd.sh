cd tools/micro && for b in walk_r_final walk_r_c0dadd walk_r_final walk_r_c0dadd; do timeout 60 ./$b; done 2>&1 | tee ../../gpurun_out/walk_exp9.log
