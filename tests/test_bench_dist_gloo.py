"""bench.py's multi-rank F_p / CRT mode (secondary.crt under torchrun), world 2 on gloo.

Each rank walks its aligned Gray share of every basis (bench.crt_section); the
walk itself is stood in for by the CPU oracle behind a Job-shaped object (no
GPU here), so the test covers the rank split, the residue gather, the Glynn
finish and the CRT lift of the bench code path: both ranks must report
perm(S_13) = 175747 (A003112) on all three bases.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _OracleJob:
    """Job.modp stand-in: residues of [start, start + length) from the oracle."""

    def __init__(self, mats, primes, algo, start, length):
        self.args = (mats, [int(p) for p in primes], algo, start, length)

    @classmethod
    def modp(cls, mats, primes, algo, start, length, device=0):
        return cls(mats, primes, algo, start, length)

    def run(self, iters=1, flush=0):
        from oracle import oracle
        mats, primes, algo, start, length = self.args
        res = [oracle.block_partial_modp(m, start, length, p, algo) for m, p in zip(mats, primes)]
        return 1.0, 1.0, res

    def groups(self):
        _, primes, _, _, _ = self.args
        return [{"kind": "reduced", "P": len(primes), "regs": 0, "ctas_per_sm": 0, "grid": 0,
                 "smem": 0, "ms": 1.0, "prime_idx": list(range(len(primes)))}]

    def close(self):
        pass


class _FakeNat:
    Job = _OracleJob


class _Args:
    crt_n = 13


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_2602_10141_b200 import dist as pkdist
    from paper_2602_10141_b200 import modular
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench._WORLD["n"] = world
    try:
        out = bench.crt_section(_Args(), _FakeNat(), modular, 148, 1965.0, rank, world, pkdist)
        q.put((rank, {k: v["value"] for k, v in out["bases"].items()}))
    finally:
        dist.destroy_process_group()


def test_crt_section_world2_gathers_to_a003112():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=240) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank in (0, 1):
        assert set(got[rank]) == {"gpu_basis", "reference_31bit", "reference_59bit_default"}
        assert all(v == "175747" for v in got[rank].values()), got[rank]
