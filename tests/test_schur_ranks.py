"""Checkpointed exact perm(S_n) across ranks (f3 on several processes), world 2 on gloo.

The GPU walk is stood in for by the CPU oracle (no GPU here), so these tests cover the
host logic of ``modular.schur_permanent_resumable`` with ``world > 1``: the chunk
deal (c = rank mod world), one checkpoint file per rank, the residue gather, resuming
with a different world size, and the file-exchange mode without a process group.
perm(S_13) = 175747 (OEIS A003112).
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_10141_b200 import modular

A003112_13 = 175747


def _oracle_walk(n, mats, primes, method, start, length, devices):
    from oracle import oracle
    return [oracle.block_partial_modp(m, start, length, int(p), method)
            for m, p in zip(mats, primes)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, ck, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2602_10141_b200 import modular as mod
    mod._schur_walk = _oracle_walk
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first = mod.schur_permanent_resumable(13, ck, chunks=8, max_chunks_this_call=1)
        second = mod.schur_permanent_resumable(13, ck, chunks=8)
        q.put((rank, first[0], first[3], second[0], second[3]))
    finally:
        dist.destroy_process_group()


def test_world2_gathers_and_resumes_on_one_rank(tmp_path, monkeypatch):
    ck = str(tmp_path / "s13.jsonl")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ck, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = {r: rest for r, *rest in (q.get(timeout=240) for _ in range(2))}
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank in (0, 1):
        v1, d1, v2, d2 = got[rank]
        assert v1 is None and d1 == 2  # one chunk per rank, gathered
        assert v2 == A003112_13 and d2 == 8
    # one writer per rank, each holding its residue class of chunks
    for rank in (0, 1):
        with open(f"{ck}.rank{rank}") as f:
            chunks = [int(x.split('"chunk": ')[1].split(",")[0]) for x in f if '"chunk"' in x]
        assert sorted(chunks) == list(range(rank, 8, 2))
    assert not os.path.exists(ck) or os.path.getsize(ck) > 0

    # a single process resumes from the rank files without walking anything
    def no_walk(*a):
        raise AssertionError("every chunk is on disk")
    monkeypatch.setattr(modular, "_schur_walk", no_walk)
    v, _, wit, done = modular.schur_permanent_resumable(13, ck, chunks=8)
    assert v == A003112_13 and done == 8 and wit


def test_file_exchange_without_a_process_group(tmp_path, monkeypatch):
    """rank/world from a scheduler, no process group: the files are the exchange."""
    monkeypatch.setattr(modular, "_schur_walk", _oracle_walk)
    ck = str(tmp_path / "s13.jsonl")
    v, _, _, done = modular.schur_permanent_resumable(13, ck, chunks=4, rank=1, world=2,
                                                      method="ryser")
    assert v is None and done == 2
    v, _, _, done = modular.schur_permanent_resumable(13, ck, chunks=4, rank=0, world=2,
                                                      method="ryser")
    assert v == A003112_13 and done == 4
    with pytest.raises(ValueError, match="different run"):
        modular.schur_permanent_resumable(13, ck, chunks=4, rank=0, world=2, method="glynn")
    with pytest.raises(ValueError, match="rank and world"):
        modular.schur_permanent_resumable(13, ck, chunks=4, rank=2, world=2)
