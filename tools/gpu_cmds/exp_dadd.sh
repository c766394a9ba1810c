cd tools/micro && for b in walk_base walk_dadd walk_r_base walk_r_dadd walk_base walk_dadd; do timeout 60 ./$b; done 2>&1 | tee ../../gpurun_out/walk_exp7.log
