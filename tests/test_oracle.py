"""The CPU oracle (oracle/ryser_oracle.c) pinned against the reference's golden vectors.

Bit-exact: every golden value came from the reference's own numba kernels
(kernels.py:33-344) via tools/make_golden.py.
"""
import numpy as np
import pytest

from conftest import bits_equal, dec_c, dec_matrix, load_golden
from oracle import oracle


@pytest.fixture(scope="module")
def f64g():
    return load_golden("f64_blocks.json")


def test_oracle_f64_blocks_bit_exact(f64g):
    assert f64g["backend"] == "numba"
    n_checked = 0
    for case in f64g["cases"]:
        a = dec_matrix(case["matrix"])
        for b in case["blocks"]:
            s, c = oracle.block_partial(a, b["start"], b["len"], case["algorithm"])
            assert bits_equal(s, dec_c(b["sum"])), (case["kind"], case["algorithm"], b)
            assert bits_equal(c, dec_c(b["comp"])), (case["kind"], case["algorithm"], b)
            n_checked += 1
    assert n_checked >= 80


def test_oracle_modp_blocks_exact():
    g = load_golden("modp_blocks.json")
    for case in g["cases"]:
        n, p = case["n"], case["p"]
        if "matrix" in case:
            a = np.array(case["matrix"], dtype=np.uint64).reshape(n, n)
        else:
            g_ = case["root"]
            pw = [pow(g_, k, p) for k in range(n)]
            a = np.array([[pw[(j * k) % n] for k in range(n)] for j in range(n)], dtype=np.uint64)
        for b in case["blocks"]:
            if case["bits"] if "bits" in case else 0:
                if case.get("bits") == 59 and b["len"] > 2000:
                    continue
            got = oracle.block_partial_modp(a, b["start"], b["len"], p, case["algorithm"])
            assert got == b["res"], (n, p, case["algorithm"], b)


def test_oracle_mulmod_against_bigint():
    rng = np.random.default_rng(5)
    for bits in (31, 59, 62):
        p = (1 << bits) - 1 if bits != 62 else (1 << 61) - 1
        for _ in range(2000):
            a, b = int(rng.integers(0, p)), int(rng.integers(0, p))
            assert oracle.mulmod(a, b, p) == a * b % p


def test_oracle_engine_combine_matches_reference_kats():
    kats = {k["tag"]: k for k in load_golden("engine_kats.json")["kats"]}
    g = load_golden("engine_kats.json")
    a = dec_matrix(g["ginibre14"])
    for blocks in (1, 7, 64):
        want = dec_c(kats[f"blocked_ginibre14_{blocks}"]["v"])
        got = oracle.permanent(a, "ryser", blocks=blocks, threads=4)
        assert bits_equal(got, want), blocks


def test_oracle_schur_values():
    g = load_golden("schur.json")
    for row in g["rows"]:
        if row["n"] > 15:
            continue
        n = row["n"]
        for p, root, res in zip(row["primes"], row["roots"], row["residues"]):
            pw = [pow(root, k, p) for k in range(n)]
            a = [[pw[(j * k) % n] for k in range(n)] for j in range(n)]
            assert oracle.permanent_modp(a, p, blocks=8) == res


def test_reference_pinned_large_schur_values_consistent():
    """The reference-produced perm(S_n), n >= 35 (tests/golden/schur_ref_large.json,
    tools/pin_schur_ref.py): the CRT lift of the reference's residues is the stored
    value, every residue is that value mod its prime, and each root is a primitive
    n-th root of unity (reference modular.py:126-147)."""
    from conftest import load_golden
    from paper_2602_10141_b200 import modular
    for row in load_golden("schur_ref_large.json")["rows"]:
        if not row.get("value"):
            continue
        n, v = row["n"], int(row["value"])
        basis = modular.find_primes(n, max_bits=31)
        assert list(basis.primes) == row["primes"]
        wit = [modular.ResidueWitness(prime=p, root=g, residue=r)
               for p, g, r in zip(row["primes"], row["roots"], row["residues"])]
        assert modular.crt_reconstruct(wit, basis) == v
        for p, g, r in zip(row["primes"], row["roots"], row["residues"]):
            assert v % p == r
            assert g == modular.primitive_nth_root(p, n)
        assert v % 2 == 1 and abs(v) <= n ** (n / 2)


@pytest.mark.parametrize("n,value", [(45, -470483360490107435783203125),
                                     (47, -52876272639843868105982022705)])
def test_schur_long_run_chunk_records(n, value):
    """The committed chunk residues of the perm(S_45) and perm(S_47) runs (tools/schur45.py):
    the chunks of each basis add up (mod p, Glynn's 2^(1-n) applied) to residues whose CRT
    lift is the recorded integer, and every extra-prime / second-basis record agrees."""
    import glob
    import json
    import math
    import os

    from paper_2602_10141_b200 import modular
    files = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", f"schur{n}_*_chunks.jsonl")))
    assert len(files) == 2
    for path in files:
        with open(path) as f:
            lines = [json.loads(x) for x in f if x.strip()]
        recs = [r for r in lines if "chunk" in r]
        assert sorted(r["chunk"] for r in recs) == list(range(64))
        if "header" in lines[0]:
            primes = lines[0]["header"]["primes"]
            tot = [sum(r["residues"][k] for r in recs) for k in range(len(primes))]
            wit = [modular.ResidueWitness(prime=p, root=0,
                                          residue=modular._schur_finish(n, t, p, "glynn"))
                   for p, t in zip(primes, tot)]
            basis = modular.CrtBasis(n, tuple(primes), math.prod(primes))
            assert modular.crt_reconstruct(wit, basis) == value
        else:  # one extra prime, named in the file
            q = int(path.rsplit("_q", 1)[1].split("_")[0])
            r = modular._schur_finish(n, sum(x["residue"] for x in recs), q, "glynn")
            assert r == value % q
    assert value % n == 0
