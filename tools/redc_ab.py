"""A/B of a Montgomery-64 walk variant against the product library (GPU box).

    PERMKIT_GPU_LIB=<variant.so> python tools/redc_ab.py n [bits]

Walks the n x n Schur residue matrix mod the largest 59-bit prime = 1 mod n (the
reference's default basis) over [0, 2^bits) and prints the per-prime result and the
rate, so two libraries can be compared for identical residues and speed.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native as nat  # noqa: E402
from tools.gpu_probe import schur_res  # noqa: E402
from tools.modp_rates import primes_desc  # noqa: E402

n = int(sys.argv[1])
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ps = primes_desc(n, 1 << 59, 1, lambda p: True)
res = np.stack([schur_res(n, p) for p in ps])
job = nat.Job.modp(res, ps, "ryser", 0, 1 << bits)
_, _, out0 = job.run(1)
_, walk, out = job.run(3)
job.close()
print(json.dumps({"lib": os.path.basename(os.environ.get("PERMKIT_GPU_LIB", "product")), "n": n,
                  "bits": bits, "prime": ps[0], "result": [int(v) for v in np.asarray(out).ravel()],
                  "ms": walk / 3, "prime_upd_per_s": n * 2.0 ** bits / (walk / 3 / 1e3)}))
