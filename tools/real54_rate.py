"""Rate of the real fp64 Glynn walk at n = 49..64 and the extrapolated time of a
full 54 x 54 real permanent ("can match [a 400-node cluster]
on a single NVIDIA GH200 in comparable wall-clock time").

    python tools/real54_rate.py [n ...]  -> one JSON line per n

The default plan walks 2^(m - 17) indices per lane (2^36 at n = 54: a full
permanent takes hours), so this samples the rate on a range of 8 waves of tiles
with $PK_PLAN_K = 20 (per-step cost does not depend on the segment length).
"""
import json
import os
import sys
import time

import numpy as np

os.environ.setdefault("PK_PLAN_K", "20")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native as nat  # noqa: E402
from paper_2602_10141_b200.ensembles import sample_matrix  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [54]:
    a = sample_matrix("ginibre-r", n, 2602, 0) / np.sqrt(n)
    k = int(os.environ["PK_PLAN_K"])
    span = (1184 * 8) << (k + 5)  # 8 waves of one tile per warp (148 SMs x 2 CTAs x 4 warps)
    job = nat.Job.f64(a, "glynn", 0, span)
    job.run(1)
    tot, walk, _ = job.run(2)
    rate = 2 * span * n / (walk / 1e3)
    full = n * 2.0 ** (n - 1) / rate
    print(json.dumps({"n": n, "algo": "glynn", "row_updates_per_s": rate, "info": job.info(),
                      "full_permanent_s": full, "full_permanent_h": full / 3600,
                      "full_permanent_h_8gpu": full / 3600 / 8}))
