"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU host logic in
paper_2507_02754_b200/parallel.py.  The compute callable is the float64 oracle here (test
infrastructure); on GPUs it is the CUDA binding.  Checks that the sequence-sharded forward and
backward with the one-step halo exchange reproduce the unsharded oracle, and that B x H
sharding partitions the slices."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_02754_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_fwd(q, k, v, k2, v2, w1, w2, n_prefix=0, det=False):
    import oracle
    o, lse = oracle.forward(q, k, v, k2, v2, w1, w2, det=det, n_prefix=n_prefix)
    return torch.from_numpy(o), torch.from_numpy(lse)


def oracle_bwd(q, k, v, k2, v2, o, lse, dO, w1, w2, n_prefix=0, det=False):
    import oracle
    g = oracle.backward(q, k, v, k2, v2, dO, w1, w2, det=det, n_prefix=n_prefix)
    return tuple(torch.from_numpy(x) for x in g)


def _worker(rank, world, port, data, w1, w2, det, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = data["q"].shape[1]
        lo, hi, _ = parallel.seq_shard(N, rank, world, max(w1, w2) - 1)
        sh = {n: torch.from_numpy(x[:, lo:hi].copy()) for n, x in data.items()}
        o, lse, ext = parallel.seq_forward(sh["q"], sh["k"], sh["v"], sh["k2"], sh["v2"], w1, w2, oracle_fwd, det=det)
        grads = parallel.seq_backward(sh["q"], ext, o, lse, sh["dO"], w1, w2, oracle_bwd, det=det)
        out[rank] = {"o": o.numpy(), "lse": lse.numpy(), "grads": [g.numpy() for g in grads]}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("world,w1,w2", [
    (2, 7, 3),   # interior queries computed while the halo is in flight (L=12 > halo 6)
    (2, 4, 9),   # w2 > w1: the K'/V' halo is the longer one
    (3, 9, 2),   # L = 8 = halo: no interior queries; the middle rank sends and receives
])
def test_sequence_sharded_matches_unsharded(oracle_mod, det, world, w1, w2):
    rng = np.random.default_rng(5)
    B, N, H, D = 1, 24, 2, 6
    data = {n: rng.standard_normal((B, N, H, D)) for n in ("q", "k", "v", "k2", "v2", "dO")}
    o_ref, lse_ref = oracle_mod.forward(data["q"], data["k"], data["v"], data["k2"], data["v2"], w1, w2, det=det)
    g_ref = oracle_mod.backward(data["q"], data["k"], data["v"], data["k2"], data["v2"], data["dO"], w1, w2, det=det)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), data, w1, w2, det, out), nprocs=world, join=True)
    L = N // world
    for r in range(world):
        sl = slice(r * L, (r + 1) * L)
        np.testing.assert_allclose(out[r]["o"], o_ref[:, sl], rtol=0, atol=1e-13)
        np.testing.assert_allclose(out[r]["lse"], lse_ref[:, :, sl], rtol=0, atol=1e-13)
        for got, ref in zip(out[r]["grads"], g_ref):
            np.testing.assert_allclose(got, ref[:, sl], rtol=0, atol=1e-12)


def test_bh_shard_partitions():
    for B, H, world in ((4, 16, 8), (8, 32, 3), (1, 5, 4), (2, 3, 8)):
        seen = []
        for r in range(world):
            lo, hi = parallel.bh_shard(B, H, r, world)
            assert 0 <= lo <= hi <= B * H
            seen.extend(range(lo, hi))
        assert seen == list(range(B * H))


def test_seq_shard_rejects_short_shards():
    with pytest.raises(ValueError):
        parallel.seq_shard(64, 1, 8, n_halo=15)
    assert parallel.seq_shard(64, 1, 4, n_halo=15) == (16, 32, 15)
    with pytest.raises(ValueError):
        parallel._check_lengths(7, 9, 2, world=2)  # queries would need rank r-2's rows
    assert parallel._check_lengths(8, 9, 2, world=2) == 8


def test_bh_slice_blocks():
    assert parallel.bh_slice(8, 32, 3, 8) == (3, 4, 0, 32)     # c5 at 8 GPUs: one batch element each
    assert parallel.bh_slice(8, 32, 1, 2) == (4, 8, 0, 32)
    assert parallel.bh_slice(4, 16, 5, 8) == (2, 3, 8, 16)     # c3 at 8 GPUs: half the heads of one b
    with pytest.raises(ValueError):
        parallel.bh_slice(3, 4, 1, 2)                           # [6, 12) spans b = 1 and 2 partially
