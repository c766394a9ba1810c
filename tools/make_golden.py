"""Generate golden fixtures from the REFERENCE implementation (run in the build container).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/make_golden.py

Imports the read-only reference package from /root/reference/pkg/src (it exists
only in the build container, never on the GPU box) and writes small JSON
fixtures to tests/golden/.  Floats are stored with float.hex() so bit-exact
comparisons survive the round trip.  The committed fixtures, not this script,
are what the tests read.
"""
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import permkit  # noqa: E402
from permkit import engine, geodesics, gray, kernels, matrices, modular  # noqa: E402
from permkit.domains import COMPLEX, INTEGER, RATIONAL, REAL, PrimeField  # noqa: E402
from permkit.ensembles import EnsembleSpec, RngStream, sample_matrix, sample_permanents  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
os.makedirs(OUT, exist_ok=True)


def hx(x):
    return float(x).hex()


def enc_matrix(a):
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return {"n": a.shape[0], "complex": True,
                "re": [hx(v) for v in a.real.ravel()], "im": [hx(v) for v in a.imag.ravel()]}
    return {"n": a.shape[0], "complex": False, "re": [hx(v) for v in a.ravel()]}


def enc_c(z):
    z = complex(z)
    return [hx(z.real), hx(z.imag)]


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, indent=0, separators=(",", ":"))
    print("wrote", name, os.path.getsize(os.path.join(OUT, name)), "bytes")


def f64_blocks():
    rnd = random.Random(2602)
    cases = []
    specs = [("haar-u", 12, 7, 0, ["ryser", "glynn"], 5000), ("haar-u", 24, 7, 0, ["ryser"], 4000),
             ("haar-u", 32, 7, 0, ["ryser"], 2500), ("ginibre-c", 16, 7, 0, ["ryser", "glynn"], 5000),
             ("haar-o", 20, 3, 1, ["ryser", "glynn"], 5000), ("goe", 10, 5, 2, ["ryser", "glynn"], 1024),
             ("gue", 9, 5, 3, ["ryser", "glynn"], 256), ("ginibre-r", 1, 1, 0, ["ryser", "glynn"], 2)]
    for kind, n, seed, idx, algos, maxlen in specs:
        a = sample_matrix(kind, n, seed, idx)
        for algo in algos:
            m = n if algo == "ryser" else n - 1
            blocks = []
            for t in range(7):
                if t == 0:
                    s, ln = 0, min(maxlen, 1 << m)
                elif t == 1:
                    s, ln = rnd.randrange(0, 1 << m), 0
                else:
                    ln = rnd.randrange(1, min(maxlen, 1 << m) + 1)
                    s = rnd.randrange(0, (1 << m) - ln + 1)
                part = kernels.ryser_partial if algo == "ryser" else kernels.glynn_partial
                sm, cm = part(a, s, ln)
                blocks.append({"start": s, "len": ln, "sum": enc_c(sm), "comp": enc_c(cm)})
            cases.append({"kind": kind, "seed": seed, "index": idx, "algorithm": algo,
                          "matrix": enc_matrix(a), "blocks": blocks})
    dump("f64_blocks.json", {"backend": kernels.backend_name(), "cases": cases})


def modp_blocks():
    rnd = random.Random(43)
    cases = []
    for n, bits, maxlen in ((24, 31, 20000), (24, 59, 1500), (36, 31, 20000), (36, 25, 20000),
                            (43, 31, 8000), (43, 59, 600), (13, 31, 8192)):
        basis = modular.find_primes(n, max_bits=bits)
        p = basis.primes[0]
        g = modular.primitive_nth_root(p, n)
        a = modular.root_matrix_mod(n, p, g)
        au = np.array([[int(x) for x in row] for row in a], dtype=np.uint64)
        for algo in ("ryser", "glynn"):
            m = n if algo == "ryser" else n - 1
            blocks = []
            for t in range(6):
                ln = rnd.randrange(1, min(maxlen, 1 << m) + 1) if t else min(maxlen, 1 << m)
                s = rnd.randrange(0, (1 << m) - ln + 1) if t else 0
                if t == 5:
                    s = (1 << m) - ln  # the top end of the range
                fn = kernels.ryser_partial_modp if algo == "ryser" else kernels.glynn_partial_modp
                blocks.append({"start": s, "len": ln, "res": fn(au, s, ln, p)})
            cases.append({"n": n, "p": p, "root": g, "bits": bits, "algorithm": algo,
                          "blocks": blocks})
    # random residue matrices, including a composite and an even modulus
    for n, p in ((20, 2147483647), (12, 15), (10, 2), (11, 4), (9, 1000003)):
        rr = np.random.default_rng(n * 31 + p)
        au = rr.integers(0, p, size=(n, n)).astype(np.uint64)
        for algo in ("ryser", "glynn"):
            m = n if algo == "ryser" else n - 1
            blocks = []
            for t in range(4):
                ln = rnd.randrange(1, min(3000, 1 << m) + 1) if t else (1 << m)
                s = rnd.randrange(0, (1 << m) - ln + 1) if t else 0
                fn = kernels.ryser_partial_modp if algo == "ryser" else kernels.glynn_partial_modp
                blocks.append({"start": s, "len": ln, "res": fn(au, s, ln, p)})
            cases.append({"n": n, "p": p, "matrix": [int(x) for x in au.ravel()],
                          "algorithm": algo, "blocks": blocks})
    dump("modp_blocks.json", {"cases": cases})


def schur():
    rows = []
    for n in range(1, 22):
        for bits in (31, 59):
            value, basis, wit = modular.schur_permanent_exact(n, max_bits=bits, threads=8)
            rows.append({"n": n, "bits": bits, "value": str(value), "primes": list(basis.primes),
                         "roots": [w.root for w in wit], "residues": [w.residue for w in wit]})
    # API helpers
    helpers = {
        "find_primes_3_asc": list(modular.find_primes(3, ascending=True).primes),
        "find_primes_20_31": list(modular.find_primes(20, max_bits=31).primes),
        "find_primes_36_31": list(modular.find_primes(36, max_bits=31).primes),
        "find_primes_43_31": list(modular.find_primes(43, max_bits=31).primes),
        "find_primes_36_59": list(modular.find_primes(36).primes),
        "root_7_3": modular.primitive_nth_root(7, 3),
        "root_13_3": modular.primitive_nth_root(13, 3),
        "root_13_3_skip1": modular.primitive_nth_root(13, 3, skip=1),
        "residue_3_7_g2": modular.schur_residue(3, 7, root=2).residue,
        "residue_2_5_g4": modular.schur_residue(2, 5, root=4).residue,
        "residue_3_13": modular.schur_residue(3, 13).residue,
        "is_prime": {str(x): modular.is_probable_prime(x) for x in
                     (1, 2, 3, 4, 97, 561, 2147483647, 2**61 - 1, 3215031751, 576460752303422617)},
        "perm_bound": {str(n): modular._perm_bound(n) for n in (1, 2, 3, 7, 10, 33)},
    }
    dump("schur.json", {"rows": rows, "helpers": helpers})


def engine_kats():
    out = []

    def rec(tag, val):
        if isinstance(val, complex):
            out.append({"tag": tag, "type": "complex", "v": enc_c(val)})
        elif isinstance(val, float):
            out.append({"tag": tag, "type": "float", "v": hx(val)})
        else:
            out.append({"tag": tag, "type": type(val).__name__, "v": str(val)})

    rec("ryser_2x2_int", permkit.perm_ryser([[1, 2], [3, 4]]))
    rec("ryser_2x2_float", permkit.perm_ryser(np.array([[1.0, 2.0], [3.0, 4.0]])))
    rec("glynn_2x2_float", permkit.perm_glynn(np.array([[1.0, 2.0], [3.0, 4.0]])))
    rec("schur3", permkit.perm_ryser(matrices.build_schur(3)))
    rec("J4", permkit.perm_ryser(matrices.build_all_ones(4)))
    rec("I7", permkit.perm_ryser(np.eye(7)))
    rec("J12_16blocks", permkit.perm_blocked(matrices.build_all_ones(12),
                                             gray.make_block_plan(12, "ryser", 16), 4))
    rec("n1_complex", permkit.perm_ryser([[2 + 3j]]))
    rec("n1_glynn_complex", permkit.perm_glynn(np.array([[2 + 3j]])))
    rec("n1_modp", permkit.perm_ryser([[7]], PrimeField(5)))
    rec("modp2_2x2", permkit.perm_ryser([[1, 2], [3, 4]], PrimeField(2)))
    rec("modp7_glynn", permkit.perm_glynn([[1, 2], [3, 4]], PrimeField(7)))
    rec("int_3x3", permkit.perm_ryser([[1, -2, 3], [4, 5, -6], [7, 8, 9]]))
    rec("int_glynn_3x3", permkit.perm_glynn([[1, -2, 3], [4, 5, -6], [7, 8, 9]]))
    from fractions import Fraction as F
    rec("rational_2x2", permkit.perm_ryser(np.array([[F(1, 2), F(1, 3)], [F(2, 5), F(3, 7)]],
                                                    dtype=object)))
    rng = np.random.default_rng(11)
    ints = rng.integers(-9, 10, size=(9, 9))
    rec("int_9x9", permkit.perm_ryser(ints.tolist()))
    rec("int_9x9_naive", permkit.perm_naive(ints.tolist()))
    rec("abs_entrywise_schur5", permkit.perm_abs_entrywise(matrices.build_schur(5)))
    rec("plan_3_2", [[b.start, b.length] for b in gray.make_block_plan(3, "ryser", 2).blocks])
    rec("plan_3_3", [[b.start, b.length] for b in gray.make_block_plan(3, "ryser", 3).blocks])
    # blocked fp64 runs with explicit plans (reference values per plan)
    a = sample_matrix("ginibre-c", 14, 5, 0)
    for blocks in (1, 7, 64):
        plan = gray.make_block_plan(14, "ryser", blocks)
        rec(f"blocked_ginibre14_{blocks}", permkit.perm_blocked(a, plan, 1))
    dump("engine_kats.json", {"kats": out, "int_9x9": ints.tolist(),
                              "ginibre14": enc_matrix(a)})


def samplers():
    out = {"matrices": [], "normals": [], "perms": []}
    for kind in ("haar-u", "haar-o", "gue", "goe", "ginibre-c", "ginibre-r"):
        for idx in (0, 3):
            out["matrices"].append({"kind": kind, "n": 5, "seed": 2602, "index": idx,
                                    "matrix": enc_matrix(sample_matrix(kind, 5, 2602, idx))})
    st = RngStream(9, 4)
    out["normals"] = [hx(v) for v in st.normals(11)]
    out["uniforms"] = [hx(v) for v in RngStream(9, 5).uniforms(5)]
    # C1: 16 Haar 20x20 with the reference engine (threads=1 -> single block)
    c1 = sample_permanents(EnsembleSpec("haar-u", 20, 16, 2602), threads=8)
    out["c1_perms"] = [enc_c(z) for z in c1]
    out["c1_first_matrix"] = enc_matrix(sample_matrix("haar-u", 20, 2602, 0))
    small = sample_permanents(EnsembleSpec("goe", 8, 20, 1), method="glynn")
    out["goe8_glynn"] = [enc_c(z) for z in small]
    dump("samplers.json", out)


def geodesic():
    out = {}
    out["cycle_7_03"] = enc_matrix(geodesics.cycle_geodesic(7, 0.3))
    out["dft_7_05"] = enc_matrix(geodesics.dft_geodesic(7, 0.5))
    out["cycle_real_7_03"] = enc_matrix(geodesics.cycle_geodesic_real(7, 0.3))
    out["cycle_real_6_03"] = enc_matrix(geodesics.cycle_geodesic_real(6, 0.3))
    for tgt in ("cycle", "dft"):
        tr = geodesics.sweep(9, tgt, 11)
        out[f"sweep_9_{tgt}"] = {"ts": [hx(t) for t in tr.ts], "perms": [enc_c(z) for z in tr.perms],
                                 "f": [hx(v) if d else None for v, d in zip(tr.f_values, tr.f_defined)]}
    tr = geodesics.sweep(8, "cycle", 5)
    out["sweep_8_cycle"] = {"perms": [enc_c(z) for z in tr.perms],
                            "defined": [bool(d) for d in tr.f_defined]}
    out["midpoint"] = {}
    for n in (5, 7, 11, 13):
        d = geodesics.midpoint_analysis(n)
        out["midpoint"][str(n)] = {"perm_mid": enc_c(d["perm_mid"]), "ratio": hx(d["ratio_to_2exp"]),
                                   "sign": d["sign"], "correction": hx(d["correction"]),
                                   "base": hx(d["cancellation_base"])}
    trd = geodesics.sweep(7, "dft", 101)
    out["recovery_7"] = hx(geodesics.recovery_ratio(trd))
    trc = geodesics.sweep(7, "cycle", 101)
    out["onset_7"] = hx(geodesics.onset_coefficient(trc))
    dump("geodesics.json", out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["f64", "modp", "schur", "engine", "samplers", "geodesic"]
    for w in which:
        {"f64": f64_blocks, "modp": modp_blocks, "schur": schur, "engine": engine_kats,
         "samplers": samplers, "geodesic": geodesic}[w]()
