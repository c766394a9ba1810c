"""perm(S_45) exactly on one B200, on two independent prime bases (checkpointed).

    python tools/schur45.py  -> gpurun_out/schur45.json, gpurun_out/s45_*.jsonl checkpoints
The paper projects ~28 GPU-hours for n = 45.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import modular  # noqa: E402


def run(tag, basis):
    t0 = time.perf_counter()
    v, b, w, done = modular.schur_permanent_resumable(45, f"gpurun_out/s45_{tag}.jsonl", chunks=16,
                                                      basis=basis)
    return {"basis": list(b.primes), "value": str(v), "chunks_done": done,
            "residues": [x.residue for x in w] if w else None,
            "wall_s": time.perf_counter() - t0}


def main():
    os.makedirs("gpurun_out", exist_ok=True)
    out = {"n": 45, "expansion": "glynn"}
    out["fast"] = run("fast", modular.gpu_prime_basis(45))
    print(json.dumps(out["fast"]), flush=True)
    out["check31"] = run("check31", modular.find_primes(45, max_bits=31))
    print(json.dumps(out["check31"]), flush=True)
    out["agree"] = out["fast"]["value"] == out["check31"]["value"]
    with open("gpurun_out/schur45.json", "w") as f:
        json.dump(out, f, indent=1)
    print("agree:", out["agree"])


if __name__ == "__main__":
    main()
