cd tools/micro && for b in walk_base walk_rot walk_r_base walk_r_rot; do timeout 60 ./$b; done 2>&1 | tee ../../gpurun_out/walk_exp5.log
