#!/bin/bash
# round 2, pass 9: full GPU suite + smoke + bench (both arms) with PAIR4 and the two-step
# Montgomery-64 body; per-group rates for the cost model; ncu of the wide walk
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c9_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c9_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c9_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c9_bench.json 2> gpurun_out/r2c9_bench.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2c9_ref.json 2> gpurun_out/r2c9_ref.err
timeout 900 python tools/modp_rates.py 32 35 36 40 --bits 34 > gpurun_out/r2c9_rates.log 2>&1
cp gpurun_out/modp_rates.json gpurun_out/r2c9_rates.json 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -c 1 -k regex:walk_modp64 -o gpurun_out/r2_wide36b python tools/prof_one.py wide 36 1 30 > gpurun_out/r2c9_ncu_wide.log 2>&1
