for n in 20 22 23 24 25 26 28; do python tools/prof_one.py batch $n 2048; done
python tools/prof_one.py batch 24 512
python tools/prof_one.py batch 24 8192
