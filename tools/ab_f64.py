"""A/B timing of the fp64 headline walk across library builds (GPU box).

    PERMKIT_GPU_LIB=<lib.so> python tools/ab_f64.py [n] [cplx] [iters]

Binds only the resident-job entry points that every build exports, so round-1
and experiment libraries (tools/build_variant.py) can be timed side by side:
walk ms per permanent of sample_matrix("haar-u"/"haar-o", n, 2602, 0).
"""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200.ensembles import sample_matrix  # noqa: E402

lib = ctypes.CDLL(os.environ["PERMKIT_GPU_LIB"])
vp, dbl = ctypes.c_void_p, ctypes.c_double
lib.pk_job_f64_create.argtypes = [ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(vp)]
lib.pk_job_run.argtypes = [vp, ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(dbl),
                           ctypes.POINTER(dbl), vp, vp]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cplx = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
a = np.ascontiguousarray(sample_matrix("haar-u" if cplx else "haar-o", n, 2602, 0))
h = vp()
assert lib.pk_job_f64_create(0, a.ctypes.data, n, cplx, 0, 0, 1 << n, ctypes.byref(h)) == 0
tot, walk = dbl(), dbl()
out = np.zeros(5)
lib.pk_job_run(h, 3, 256 << 20, ctypes.byref(tot), ctypes.byref(walk), out.ctypes.data, None)
lib.pk_job_run(h, iters, 256 << 20, ctypes.byref(tot), ctypes.byref(walk), out.ctypes.data, None)
ms = walk.value / iters
print(json.dumps({"lib": os.path.basename(os.environ["PERMKIT_GPU_LIB"]), "n": n, "cplx": cplx,
                  "walk_ms": ms, "upd_per_s": n * 2.0 ** n / (ms / 1e3),
                  "perm": [out[0] + out[1], out[2] + out[3]]}))
