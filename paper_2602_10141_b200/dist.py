"""Multi-process (one rank per GPU) sharding of the Gray walk.

The walk shards without any data-path exchange: rank r of W owns
the aligned Gray range [r 2^m / W, (r+1) 2^m / W) of one permanent (or a
contiguous slice of a batch).  The only exchange is the final gather of a
handful of scalars per rank:

* fp64: each rank returns its compensated (sum, comp) pair, the root of its
  subtree of the device-independent reduction tree (csrc/pk_reduce.cuh); the
  pairs are combined here with the same TwoSum node rule in a binary tree, so
  a power-of-two world reproduces the single-GPU bits exactly;
* F_p: residues are summed mod p (exact, order-free).

torch.distributed is plumbing only (all_gather_object over NCCL or gloo).
"""

from __future__ import annotations


def _two_sum_node(a_s, a_c, b_s, b_c):
    s = a_s + b_s
    bp = s - a_s
    ap = s - bp
    e = (a_s - ap) + (b_s - bp)
    return s, (a_c + b_c) + e


def pair_combine(a, b):
    """Combine two compensated pairs (sum, comp); complex values per component.

    Same operation order as pk::pair_combine (csrc/pk_common.cuh).
    """
    (as_, ac), (bs, bc) = a, b
    if isinstance(as_, complex) or isinstance(bs, complex):
        as_, ac, bs, bc = complex(as_), complex(ac), complex(bs), complex(bc)
        sr, cr = _two_sum_node(as_.real, ac.real, bs.real, bc.real)
        si, ci = _two_sum_node(as_.imag, ac.imag, bs.imag, bc.imag)
        return complex(sr, si), complex(cr, ci)
    return _two_sum_node(float(as_), float(ac), float(bs), float(bc))


def combine_pairs(parts):
    """Binary tree over a power-of-two list of pairs (else a left fold), as the
    library combines its per-device roots (pk_capi.cu combine_roots)."""
    cur = list(parts)
    if not cur:
        return 0.0, 0.0
    if len(cur) & (len(cur) - 1) == 0:
        while len(cur) > 1:
            cur = [pair_combine(cur[i], cur[i + 1]) for i in range(0, len(cur), 2)]
        return cur[0]
    acc = cur[0]
    for p in cur[1:]:
        acc = pair_combine(acc, p)
    return acc


def shard_range(m: int, rank: int, world: int):
    """(start, length) of rank's aligned share of [0, 2^m); world must be a power of two."""
    if world < 1 or world & (world - 1):
        raise ValueError("world size must be a power of two for an aligned Gray split")
    if world > (1 << m):
        raise ValueError("more ranks than Gray indices")
    span = (1 << m) // world
    return rank * span, span


def shard_slice(count: int, rank: int, world: int):
    """Contiguous [lo, hi) slice of a batch of ``count`` items for ``rank``."""
    return count * rank // world, count * (rank + 1) // world


def gather_pairs(local_pair, group=None):
    """All-gather every rank's (sum, comp) and combine them in rank order."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, local_pair, group=group)
    return combine_pairs(parts)


def gather_residues(local_residues, primes, group=None):
    """All-gather per-rank residue lists and add them mod p."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, [int(r) for r in local_residues], group=group)
    return [sum(p[k] for p in parts) % int(q) for k, q in enumerate(primes)]
