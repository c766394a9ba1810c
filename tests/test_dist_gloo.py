"""World-size-2 gloo runs of the rank sharding + gather logic (CPU only).

Each rank walks its aligned Gray share with the CPU oracle (standing in for the
rank's GPU); the gather must reproduce the single-process combination exactly
(F_p: the full-range residue; fp64: the same tree combine of the same pairs).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_10141_b200 import dist as pkdist
from paper_2602_10141_b200 import modular


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 14
        p = modular.gpu_prime_basis(n).primes[0]
        a = modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n))
        st, ln = pkdist.shard_range(n, rank, world)
        r = oracle.block_partial_modp(a, st, ln, p)
        total = pkdist.gather_residues([r], [p])
        rng = np.random.default_rng(0)
        m = rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12))
        st, ln = pkdist.shard_range(12, rank, world)
        pair = oracle.block_partial(m, st, ln)
        combined = pkdist.gather_pairs(pair)
        if rank == 0:
            q.put((total, combined))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_and_gather():
    from oracle import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    total, combined = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    n = 14
    p = modular.gpu_prime_basis(n).primes[0]
    a = modular._root_matrix_u64(n, p, modular.primitive_nth_root(p, n))
    assert total == [oracle.block_partial_modp(a, 0, 1 << n, p)]
    rng = np.random.default_rng(0)
    m = rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12))
    parts = [oracle.block_partial(m, 0, 2048), oracle.block_partial(m, 2048, 2048)]
    assert combined == pkdist.combine_pairs(parts)
    full = oracle.block_partial(m, 0, 4096)
    assert abs((combined[0] + combined[1]) - (full[0] + full[1])) < 1e-12 * abs(full[0])


def test_shard_helpers():
    assert pkdist.shard_range(10, 3, 4) == (768, 256)
    with pytest.raises(ValueError):
        pkdist.shard_range(10, 0, 3)
    assert [pkdist.shard_slice(10, r, 3) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
    assert pkdist.combine_pairs([(1.0, 0.0), (1e-20, 0.0)]) == (1.0, 1e-20)
