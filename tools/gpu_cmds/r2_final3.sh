#!/bin/bash
# round 2 re-entry: column-sum Montgomery-64 REDC (PK_REDC64_PS) adopted; wide parity first, then the
# full GPU suite, smoke, both bench arms, and the Montgomery-64 rates
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "wide or schur_default or 59" > gpurun_out/r2f3_wide.txt 2>&1
echo "pytest wide rc=$?" >> gpurun_out/r2f3_wide.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f3_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f3_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f3_smoke.txt 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f3_bench.json 2> gpurun_out/r2f3_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f3_ref.json 2> gpurun_out/r2f3_ref.err
timeout 600 python tools/modp_rates.py 32 35 36 --bits 34 --only wide1 wide2 --out gpurun_out/modp_rates_ps.json > gpurun_out/modp_rates_ps.log 2>&1
