"""Multi-GPU plumbing for sliding-window 2-simplicial attention.

Two modes, one process per GPU (torch.distributed; NCCL on GPUs, gloo in the CPU tests):

* B x H sharding (`bh_shard`, `bh_slice`): every (b, h) slice is independent (the kernels'
  grid axis), so rank r takes a contiguous range of the B*H slices and no data-path collective
  exists.

* Sequence sharding (`seq_forward` / `seq_backward`): rank r owns the query rows
  [r*L, (r+1)*L) of every (b, h) and the key rows with the same positions.  A query at position
  pos needs key rows (pos-w1, pos] of K, V and (pos-w2, pos] of K', V', so before the forward each
  rank sends its last w1-1 rows of k, v and its last w2-1 rows of k2, v2 to rank r+1 (one
  `batch_isend_irecv` group) and calls the kernel with n_prefix = max(w1, w2) - 1 (the shorter
  halo is zero-padded in front: those rows lie outside every window and are never read).  The
  interior queries (local i >= n_prefix) need no halo: they run while the exchange is in flight,
  and only the n_prefix boundary queries wait for it.  In the backward the gradients of the halo
  rows are partial sums owned by rank r-1: they travel back (r -> r-1) and are added there.
  Rank 0 has no predecessor (the chain is not a ring).

The compute itself is a callable with the signature of `binding.forward` / `binding.backward`
(the CUDA library in production).  Only this file's exchange logic runs on the host; the
concatenations and additions below are data movement of the plumbing, not the method.
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


def bh_slice(B: int, H: int, rank: int, world: int):
    """The rank's B x H shard as a rectangular block of a [B, N, H, D] tensor:
    (b0, b1, h0, h1) with the flat range of `bh_shard` = whole batch elements [b0, b1) (all heads)
    or heads [h0, h1) of one batch element.  Raises if the flat range is neither."""
    lo, hi = bh_shard(B, H, rank, world)
    if lo % H == 0 and hi % H == 0:
        return lo // H, hi // H, 0, H
    if lo // H == (hi - 1) // H:
        return lo // H, lo // H + 1, lo % H, (hi - 1) % H + 1
    raise ValueError(f"B={B} H={H} over {world} ranks: rank {rank}'s slices [{lo}, {hi}) span a batch "
                     "boundary; choose a world size dividing B or B*H/world dividing H")


def seq_shard(N: int, rank: int, world: int, n_halo: int):
    """Query range [lo, hi) of `rank` and the prefix length it receives."""
    if N % world != 0:
        raise ValueError("sequence length must divide evenly across ranks")
    L = N // world
    lo = rank * L
    if world > 1 and L < n_halo:
        raise ValueError(f"shard length {L} shorter than the halo {n_halo}: use fewer ranks")
    return lo, lo + L, (min(n_halo, lo) if rank > 0 else 0)


def _halo_sizes(w1: int, w2: int):
    return w1 - 1, w2 - 1, max(w1, w2) - 1


def _start_forward_exchange(k, v, k2, v2, w1: int, w2: int, rank: int, world: int, group=None):
    """Post the halo sends (last w1-1 rows of k, v; last w2-1 of k2, v2) to rank+1 and the matching
    receives from rank-1.  Returns (requests, received buffers or [])."""
    h1, h2, _ = _halo_sizes(w1, w2)
    ops, recv = [], []
    sizes = (h1, h1, h2, h2)
    if rank + 1 < world:
        for t, n in zip((k, v, k2, v2), sizes):
            if n > 0:
                ops.append(dist.P2POp(dist.isend, t[:, -n:].contiguous(), rank + 1, group))
    if rank > 0:
        for t, n in zip((k, v, k2, v2), sizes):
            buf = torch.empty((t.shape[0], n) + tuple(t.shape[2:]), dtype=t.dtype, device=t.device)
            recv.append(buf)
            if n > 0:
                ops.append(dist.P2POp(dist.irecv, buf, rank - 1, group))
    reqs = dist.batch_isend_irecv(ops) if ops else []
    return reqs, recv


def _pad_front(t, n: int):
    """[B, m, H, D] -> [B, n, H, D] with zero rows in front (rows outside every window)."""
    if t.shape[1] == n:
        return t
    z = torch.zeros((t.shape[0], n - t.shape[1]) + tuple(t.shape[2:]), dtype=t.dtype, device=t.device)
    return torch.cat([z, t], dim=1)


def _check_lengths(L: int, w1: int, w2: int, world: int):
    n_halo = max(w1, w2) - 1
    if world > 1 and L < max(n_halo, 1):
        raise ValueError(f"local sequence length {L} shorter than the halo {n_halo} "
                         f"(max(w1, w2) - 1): queries would need rows from rank r-2; use fewer ranks")
    return n_halo


def seq_forward(q, k, v, k2, v2, w1: int, w2: int, fwd: Callable, group=None, **kw):
    """Sequence-sharded forward.  q/k/v/k2/v2 are this rank's [B, L, H, D] shards.
    Returns (o, lse) for the local queries and the context seq_backward needs."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    L = q.shape[1]
    n_halo = _check_lengths(L, w1, w2, world)
    reqs, halos = _start_forward_exchange(k, v, k2, v2, w1, w2, rank, world, group) if n_halo > 0 \
        else ([], [])
    split = rank > 0 and n_halo > 0 and n_halo < L
    if split:
        # interior queries [n_halo, L): their windows lie inside the local keys (first n_halo local
        # rows as prefix) -- computed while the halo is in flight
        o_in, lse_in = fwd(q[:, n_halo:].contiguous(), k, v, k2, v2, w1, w2, n_prefix=n_halo, **kw)
    for r in reqs:
        r.wait()
    if rank > 0 and n_halo > 0:
        hk, hv, hk2, hv2 = (_pad_front(h, n_halo) for h in halos)
        nb = n_halo if split else L  # boundary queries
        keys = tuple(torch.cat([hb, t[:, :nb]], dim=1) for hb, t in zip((hk, hv, hk2, hv2), (k, v, k2, v2)))
        o_b, lse_b = fwd(q[:, :nb].contiguous(), *keys, w1, w2, n_prefix=n_halo, **kw)
        if split:
            o = torch.cat([o_b, o_in], dim=1)
            lse = torch.cat([lse_b, lse_in], dim=2)
        else:
            o, lse = o_b, lse_b
        ctx = (k, v, k2, v2, (hk, hv, hk2, hv2), n_halo, split)
    else:
        o, lse = fwd(q, k, v, k2, v2, w1, w2, n_prefix=0, **kw)
        ctx = (k, v, k2, v2, None, 0, False)
    return o, lse, ctx


def seq_backward(q, ctx, o, lse, dO, w1: int, w2: int, bwd: Callable, group=None, **kw):
    """Sequence-sharded backward.  `ctx` is seq_forward's context.  Returns this rank's complete
    (dq, dk, dv, dk2, dv2) for its own L query / key rows."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    k, v, k2, v2, halos, n_halo, split = ctx
    L = q.shape[1]
    h1, h2, nh_full = _halo_sizes(w1, w2)
    if halos is None:
        dq, *kg = bwd(q, k, v, k2, v2, o, lse, dO, w1, w2, n_prefix=0, **kw)
        halo_g = None
    else:
        nb = n_halo if split else L
        keys = tuple(torch.cat([hb, t[:, :nb]], dim=1) for hb, t in zip(halos, (k, v, k2, v2)))
        g_b = bwd(q[:, :nb].contiguous(), *keys, o[:, :nb].contiguous(), lse[:, :, :nb].contiguous(),
                  dO[:, :nb].contiguous(), w1, w2, n_prefix=n_halo, **kw)
        halo_g = [g[:, :n_halo] for g in g_b[1:]]
        if split:
            g_in = bwd(q[:, nb:].contiguous(), k, v, k2, v2, o[:, nb:].contiguous(), lse[:, :, nb:].contiguous(),
                       dO[:, nb:].contiguous(), w1, w2, n_prefix=n_halo, **kw)
            dq = torch.cat([g_b[0], g_in[0]], dim=1)
            kg = [gi.clone() for gi in g_in[1:]]
            for gi, gb in zip(kg, g_b[1:]):
                gi[:, :nb] += gb[:, n_halo:]
        else:
            dq = g_b[0]
            kg = [gb[:, n_halo:].contiguous() for gb in g_b[1:]]
    # partial gradients of the halo rows go back to their owner (rank-1): the last w1-1 rows of
    # dk, dv and the last w2-1 rows of dk2, dv2 (the rows the halo actually carried)
    sizes = (h1, h1, h2, h2)
    ops, recv = [], []
    if halo_g is not None:
        for g, n in zip(halo_g, sizes):
            if n > 0:
                ops.append(dist.P2POp(dist.isend, g[:, n_halo - n:].contiguous(), rank - 1, group))
    if rank + 1 < world and nh_full > 0:
        for g, n in zip(kg, sizes):
            buf = torch.empty((g.shape[0], n) + tuple(g.shape[2:]), dtype=g.dtype, device=g.device)
            recv.append(buf)
            if n > 0:
                ops.append(dist.P2POp(dist.irecv, buf, rank + 1, group))
    for r in (dist.batch_isend_irecv(ops) if ops else []):
        r.wait()
    if recv:
        kg = [g if g.is_contiguous() else g.contiguous() for g in kg]
        for g, r_, n in zip(kg, recv, sizes):
            if n > 0:
                g[:, L - n:] += r_
    return (dq, *kg)
