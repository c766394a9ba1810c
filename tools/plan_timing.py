"""perm_blocked at the plan level vs a full perm_ryser.

    python tools/plan_timing.py [n] [blocks] -> one JSON line

Times (wall, after a warm-up call, best of 5) engine.perm_ryser(a) and
engine.perm_blocked(a, make_block_plan(n, "ryser", blocks)) on the same
matrix; the plan's blocks are unaligned (2^n / blocks is not a tile multiple),
so every block has ragged pieces.  Round 1 made one C-ABI round trip per block.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import engine  # noqa: E402
from paper_2602_10141_b200.ensembles import sample_matrix  # noqa: E402
from paper_2602_10141_b200.gray import make_block_plan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 512
a = sample_matrix("haar-u", n, 2602, 0)
plan = make_block_plan(n, "ryser", blocks)


def best(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        v = fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), v


t_full, v_full = best(lambda: engine.perm_ryser(a))
t_plan, v_plan = best(lambda: engine.perm_blocked(a, plan))
print(json.dumps({"n": n, "blocks": blocks, "perm_ryser_s": t_full, "perm_blocked_s": t_plan,
                  "ratio": t_plan / t_full, "rel_diff": abs(v_plan - v_full) / abs(v_full)}))
