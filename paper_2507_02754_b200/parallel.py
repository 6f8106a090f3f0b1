"""Multi-GPU plumbing for sliding-window 2-simplicial attention.

Two modes, one process per GPU (torch.distributed; NCCL on GPUs, gloo in the CPU tests):

* B x H sharding (`bh_shard`): every (b, h) slice is independent (the kernels' grid axis),
  so rank r takes a contiguous range of the B*H slices and no data-path collective exists.

* Sequence sharding (`seq_forward` / `seq_backward`): rank r owns the query rows
  [r*L, (r+1)*L) of every (b, h) and the key rows with the same positions.  A query at position
  pos needs key rows (pos-w, pos], so before the forward each rank sends its last
  n_halo = max(w1, w2) - 1 key rows (k, v, k2, v2) to rank r+1 (one `batch_isend_irecv` group)
  and calls the kernel with n_prefix = n_halo.  In the backward the gradients of those halo rows
  are partial sums owned by rank r-1: they travel back (r -> r-1) and are added there.  Rank 0
  has no predecessor (the chain is not a ring).

The compute itself is a callable with the signature of `binding.forward` / `binding.backward`
(the CUDA library in production).  Only this file's exchange logic runs on the host.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def bh_shard(B: int, H: int, rank: int, world: int):
    """Contiguous range [lo, hi) of flat b*H+h slices owned by `rank` (balanced, deterministic)."""
    total = B * H
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def seq_shard(N: int, rank: int, world: int, n_halo: int):
    """Query range [lo, hi) of `rank` and the prefix length it receives."""
    assert N % world == 0, "sequence length must divide evenly across ranks"
    L = N // world
    lo = rank * L
    if rank > 0 and L < n_halo:
        raise ValueError(f"shard length {L} shorter than the halo {n_halo}: use fewer ranks")
    return lo, lo + L, (min(n_halo, lo) if rank > 0 else 0)


def _exchange_forward(tensors, n_halo: int, rank: int, world: int, group=None):
    """Send the last n_halo rows (dim 1) of each tensor to rank+1; receive rank-1's.
    Returns the received halos (list, empty on rank 0)."""
    ops, recv = [], []
    if rank + 1 < world:
        for t in tensors:
            ops.append(dist.P2POp(dist.isend, t[:, -n_halo:].contiguous(), rank + 1, group))
    if rank > 0:
        for t in tensors:
            buf = torch.empty((t.shape[0], n_halo) + tuple(t.shape[2:]), dtype=t.dtype, device=t.device)
            recv.append(buf)
            ops.append(dist.P2POp(dist.irecv, buf, rank - 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return recv


def seq_forward(q, k, v, k2, v2, w1: int, w2: int, fwd: Callable, group=None, **kw):
    """Sequence-sharded forward.  q/k/v/k2/v2 are this rank's [B, L, H, D] shards.
    Returns (o, lse) for the local queries and the halo-extended key tensors (for the backward)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n_halo = max(w1, w2) - 1
    halos = _exchange_forward((k, v, k2, v2), n_halo, rank, world, group) if n_halo > 0 else []
    if halos:
        k, v, k2, v2 = (torch.cat([hb, t], dim=1) for hb, t in zip(halos, (k, v, k2, v2)))
        n_prefix = n_halo
    else:
        n_prefix = 0
    o, lse = fwd(q, k, v, k2, v2, w1, w2, n_prefix=n_prefix, **kw)
    return o, lse, (k, v, k2, v2, n_prefix)


def seq_backward(q, ext, o, lse, dO, w1: int, w2: int, bwd: Callable, group=None, **kw):
    """Sequence-sharded backward.  `ext` is seq_forward's (k, v, k2, v2, n_prefix).  Returns this
    rank's complete (dq, dk, dv, dk2, dv2) for its own L key rows."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    k, v, k2, v2, n_prefix = ext
    grads = bwd(q, k, v, k2, v2, o, lse, dO, w1, w2, n_prefix=n_prefix, **kw)
    dq, key_grads = grads[0], list(grads[1:])
    n_halo = max(w1, w2) - 1
    # partial gradients of the halo rows go back to their owner (rank-1); ours come from rank+1
    ops, recv = [], []
    if rank > 0 and n_prefix > 0:
        for g in key_grads:
            ops.append(dist.P2POp(dist.isend, g[:, :n_prefix].contiguous(), rank - 1, group))
    if rank + 1 < world and n_halo > 0:
        for g in key_grads:
            buf = torch.empty((g.shape[0], n_halo) + tuple(g.shape[2:]), dtype=g.dtype, device=g.device)
            recv.append(buf)
            ops.append(dist.P2POp(dist.irecv, buf, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    own = [g[:, n_prefix:] for g in key_grads]
    if recv:
        own = [g.clone() for g in own]
        for g, r in zip(own, recv):
            g[:, -n_halo:] += r
    return (dq, *own)
