"""Pin perm(S_n) for large odd n with the REFERENCE's own CPU path (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache nice python tools/pin_schur_ref.py 35 [threads] [glynn]

Runs `modular.schur_residue(n, p, threads=T)` (reference `modular.py:160-170`: the blocked
Ryser engine over GF(p), numba kernels `kernels.py:250-290`) for every prime of
`find_primes(n, max_bits=31)` (`modular.py:95-112`), then `crt_reconstruct` (`:173-185`).
With "glynn" each residue comes from the reference's public perm_blocked over a
Glynn block plan (engine.py:273-279, 213-258, numba kernels.py:293-344; half of
Ryser's 2^n steps) on the same root matrix (modular.py:150-157) and prime.
Each finished residue is appended to tests/golden/schur_ref_large.json immediately, so a
cut-off run keeps what it finished; a restart skips primes already recorded.  The committed
JSON, not this script, is what the GPU tests read (the reference does not exist on the box).
"""
import json
import os
import sys
import time

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from permkit import engine, gray, modular  # noqa: E402
from permkit.domains import PrimeField  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden", "schur_ref_large.json")


def load():
    if os.path.exists(OUT):
        with open(OUT) as f:
            return json.load(f)
    return {"source": "reference permkit modular.schur_residue (Ryser, GF(p), numba), "
                      "find_primes(n, max_bits=31), crt_reconstruct; tools/pin_schur_ref.py",
            "rows": []}


def save(doc):
    tmp = OUT + ".tmp"
    with open(tmp, "w") as f:
        json.dump(doc, f, indent=1)
    os.replace(tmp, OUT)


def main():
    n = int(sys.argv[1])
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    method = sys.argv[3] if len(sys.argv) > 3 else "ryser"
    basis = modular.find_primes(n, max_bits=31)
    doc = load()
    row = next((r for r in doc["rows"] if r["n"] == n and r["bits"] == 31), None)
    if row is None:
        row = {"n": n, "bits": 31, "primes": list(basis.primes), "roots": [], "residues": [],
               "seconds": [], "threads": threads, "method": method, "value": None}
        doc["rows"].append(row)
    for p in basis.primes[len(row["residues"]):]:
        t0 = time.perf_counter()
        if method == "glynn":
            g = modular.primitive_nth_root(p, n)
            a = modular.root_matrix_mod(n, p, g)
            plan = gray.make_block_plan(n, gray.GLYNN, min(64 * threads, 1 << (n - 1)))
            r = engine.perm_blocked(a, plan, worker_count=threads, domain=PrimeField(p))
            w = modular.ResidueWitness(prime=p, root=g, residue=int(r))
        else:
            w = modular.schur_residue(n, p, threads=threads)
        dt = time.perf_counter() - t0
        row["roots"].append(w.root)
        row["residues"].append(w.residue)
        row["seconds"].append(round(dt, 1))
        save(doc)
        print(f"n={n} p={p} g={w.root} r={w.residue} {dt:.0f}s", flush=True)
    wit = [modular.ResidueWitness(prime=p, root=g, residue=r)
           for p, g, r in zip(row["primes"], row["roots"], row["residues"])]
    row["value"] = str(modular.crt_reconstruct(wit, basis))
    save(doc)
    print(f"perm(S_{n}) = {row['value']}", flush=True)


if __name__ == "__main__":
    main()
