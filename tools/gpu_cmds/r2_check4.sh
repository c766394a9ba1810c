#!/bin/bash
# round 2, pass 4: full GPU suite + smoke + bench (both arms) on the pass-3 fixes
# (column-0 layout, plan fold in C, mix ceilings); plan timing
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c4_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c4_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c4_smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2c4_bench.json 2> gpurun_out/r2c4_bench.err
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2c4_ref.json 2> gpurun_out/r2c4_ref.err
for nb in "24 512" "28 512" "20 64" "32 1024"; do timeout 120 python tools/plan_timing.py $nb >> gpurun_out/r2c4_plan_timing.txt 2>&1; done
