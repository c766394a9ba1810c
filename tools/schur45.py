"""perm(S_45) exactly on one B200, on two independent prime bases (checkpointed).

    python tools/schur45.py  -> gpurun_out/schur45.json, gpurun_out/s45_*.jsonl checkpoints
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/schur45.py   (one rank per GPU)
Under torchrun each rank walks chunks c = rank (mod world) on its own GPU
(set_device_base(LOCAL_RANK)), writes s45_*.jsonl.rank<r>, and the residues are
gathered over a gloo group; a rerun with any world size resumes from all the files.
The paper projects ~28 GPU-hours for n = 45.
$S45_CHECK=59 checks on the reference's default 59-bit basis (Montgomery-64 walks);
$S45_CHECK=prime replaces the second full basis by one extra 31-bit prime q outside the
first basis (chunked and checkpointed too): value mod q must equal the walked residue.
$S45_N picks another odd n (a quick multi-rank check: S45_N=33 PK_LOGICAL_DEVICES=2
torchrun --nproc-per-node 2 ... runs two ranks on one GPU, each on its own context).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10141_b200 import _native, modular  # noqa: E402

CKDIR = os.environ.get("S45_CKDIR", "gpurun_out")  # copy checkpoints here to resume a cut run
N = int(os.environ.get("S45_N", "45"))
CHUNKS = 64  # 2^44 / 64 = 2^38 Glynn indices per chunk: 8 ranks get 8 chunks each


def run(tag, basis):
    t0 = time.perf_counter()
    v, b, w, done = modular.schur_permanent_resumable(N, os.path.join(CKDIR, f"s{N}_{tag}.jsonl"),
                                                      chunks=CHUNKS, basis=basis)
    return {"basis": list(b.primes), "value": str(v), "chunks_done": done,
            "residues": [x.residue for x in w] if w else None,
            "wall_s": time.perf_counter() - t0}


def check_prime(q, value):
    """perm(S_N) mod q by the same chunked Glynn walk, against value mod q."""
    t0 = time.perf_counter()
    ck = os.path.join(CKDIR, f"s{N}_q{q}.jsonl")
    g = modular.primitive_nth_root(q, N)
    mats = np.stack([modular._root_matrix_u64(N, q, g)])
    done = {}
    if os.path.exists(ck):
        with open(ck) as f:
            done = {r["chunk"]: r["residue"] for r in map(json.loads, f) if r}
    span = (1 << (N - 1)) // CHUNKS
    for c in range(CHUNKS):
        if c in done:
            continue
        done[c] = int(modular._schur_walk(N, mats, [q], "glynn", c * span, span, None)[0])
        with open(ck, "a") as f:
            f.write(json.dumps({"chunk": c, "residue": done[c]}) + "\n")
    res = modular._schur_finish(N, sum(done.values()), q, "glynn")
    return {"prime": q, "root": g, "residue": res, "value_mod_q": value % q,
            "agree": res == value % q, "wall_s": time.perf_counter() - t0}


def main():
    os.makedirs("gpurun_out", exist_ok=True)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        _native.set_device_base(int(os.environ.get("LOCAL_RANK", "0")))
    out = {"n": N, "expansion": "glynn", "world": world}
    out["fast"] = run("fast", modular.gpu_prime_basis(N))
    print(json.dumps(out["fast"]), flush=True)
    if os.environ.get("S45_CHECK") == "prime":
        fast = set(out["fast"]["basis"])
        q = next(p for p in modular.find_primes(N, max_bits=31).primes if p not in fast)
        out["check_prime"] = check_prime(q, int(out["fast"]["value"]))
        print(json.dumps(out["check_prime"]), flush=True)
        out["agree"] = out["check_prime"]["agree"]
    elif os.environ.get("S45_CHECK") == "59":  # the reference's default basis (modular.py:25)
        out["check59"] = run("check59", modular.find_primes(N, max_bits=59))
        print(json.dumps(out["check59"]), flush=True)
        out["agree"] = out["fast"]["value"] == out["check59"]["value"]
    else:
        out["check31"] = run("check31", modular.find_primes(N, max_bits=31))
        print(json.dumps(out["check31"]), flush=True)
        out["agree"] = out["fast"]["value"] == out["check31"]["value"]
    if int(os.environ.get("RANK", "0")) == 0:
        tag = os.environ.get("S45_CHECK", "")
        with open(f"gpurun_out/schur{N}_w{world}{'_' + tag if tag else ''}.json"
                  if (N != 45 or tag) else "gpurun_out/schur45.json", "w") as f:
            json.dump(out, f, indent=1)
        print("agree:", out["agree"])


if __name__ == "__main__":
    main()
