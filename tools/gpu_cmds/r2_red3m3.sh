#!/bin/bash
# reduced Montgomery-32 walks at 3 CTAs/SM (PK_MINCTA_T=128, spills 36-68 B) vs the product (2 CTAs/SM)
mkdir -p gpurun_out
timeout 600 python tools/modp_rates.py 33 35 --bits 34 --only red3 red2 > gpurun_out/r2m_base.txt 2>&1; echo base rc=$?
cp gpurun_out/modp_rates.json gpurun_out/r2m_base.json
PERMKIT_GPU_LIB=paper_2602_10141_b200/_lib_var/red3m3.so timeout 600 python tools/modp_rates.py 33 35 --bits 34 --only red3 red2 > gpurun_out/r2m_m3.txt 2>&1; echo m3 rc=$?
cp gpurun_out/modp_rates.json gpurun_out/r2m_m3.json
