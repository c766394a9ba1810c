#!/bin/bash
# round 2: C4 (perm(S_n), n = 35..43 on the final build, n = 37 / 39 cross-checked on the
# reference's 31-bit basis with Ryser) and the full-size C2 / C5 configs
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python tools/schur_run.py 35 37 39 41 43 --check 37 39 --out gpurun_out/r2_schur_c4.json > gpurun_out/r2_schur_c4.log 2>&1
timeout 600 python tools/configs_run.py > gpurun_out/r2_configs_full.jsonl 2> gpurun_out/r2_configs_full.err
