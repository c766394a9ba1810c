# headline bench + launch list + ncu --set full captures of the walk kernels (one GPU)
timeout 900 python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1e.csv python bench.py --steps 2 --warmup 1 --no-secondary > gpurun_out/ncu_launch_r1e.log 2>&1
for spec in "f64c 32" "f64r 32" "basis 36" "hyb 36" "wide 32"; do
  set -- $spec
  timeout 600 python tools/prof_one.py $1 $2 > gpurun_out/plain_$1_$2.log 2>&1 || continue
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_ -c 1 -f -o gpurun_out/prof_r1e_$1$2 python tools/prof_one.py $1 $2 > gpurun_out/ncu_r1e_$1$2.log 2>&1
done
tail -c 1500 gpurun_out/bench_r1e.json; cat gpurun_out/plain_*.log
