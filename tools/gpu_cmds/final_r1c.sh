timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_final3.log 2>&1; tail -3 gpurun_out/gpu_final3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final3.log 2>&1; tail -1 gpurun_out/smoke_final3.log
timeout 900 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; tail -c 1200 gpurun_out/bench_final3.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final3.csv python bench.py --steps 2 --warmup 1 --no-secondary > gpurun_out/ncu_launch_final3.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:walk_ -c 1 -f -o gpurun_out/prof_final3_f64c32 python tools/prof_one.py f64c 32 > gpurun_out/ncu_final3_f64c32.log 2>&1; tail -1 gpurun_out/ncu_final3_f64c32.log
timeout 2400 python tools/schur_run.py 35 36 37 39 41 43 --check 39 --out gpurun_out/schur_final3.json > gpurun_out/schur_final3.log 2>&1; cut -c1-200 gpurun_out/schur_final3.log
