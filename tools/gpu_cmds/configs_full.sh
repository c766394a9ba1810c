# full-size C2 (Haar n=23 x 50,000) and C5 (n = 28) through the public API
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv > gpurun_out/cfg_smi.log
nproc >> gpurun_out/cfg_smi.log
timeout 1200 python tools/configs_run.py > gpurun_out/configs_full.jsonl 2> gpurun_out/configs_full.err; cat gpurun_out/configs_full.jsonl; tail -3 gpurun_out/configs_full.err
