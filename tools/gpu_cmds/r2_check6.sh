#!/bin/bash
# round 2, pass 6: the bench's N > 1 path (2 ranks sharing the GPU over gloo), the
# round-2 launch list of the bench, ncu of the headline and the n = 54 real walk,
# and the full GPU suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
PK_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2c6_bench_n2.json 2> gpurun_out/r2c6_bench_n2.err
echo "n2 rc=$?" >> gpurun_out/r2c6_bench_n2.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c6_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c6_pytest.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2c6_ncu_bench.log 2>&1
NCU="ncu --set full --import-source on --clock-control none -c 1"
timeout 600 $NCU -k regex:walk_f64 -o gpurun_out/r2_f64c32 python tools/prof_one.py f64c 32 1 > gpurun_out/r2c6_ncu_f64c.log 2>&1
PK_PLAN_K=16 timeout 600 $NCU -k regex:walk_f64 -o gpurun_out/r2_f64r54 python tools/real54_rate.py 54 > gpurun_out/r2c6_ncu_real54.log 2>&1
