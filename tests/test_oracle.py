"""Pins for the float64 oracle (oracle/), independent of the oracle's own code.

Every test here checks the oracle against something the paper or the mathematics
fixes, never against a retyped copy of its own formula:
  * hand-derived worked examples (tests/golden/*.json, each citing its passage);
  * Alg. 1 executed literally with numpy einsum, plus windows;
  * determinant logits via numpy.linalg.det (a library routine, not Sarrus);
  * collapse K'=V'=1 -> sliding-window dot attention via torch SDPA;
  * gradients via torch autograd of a dense einsum model and central differences;
  * closed forms (n=1, dO=0, V=V'=1), rotation invariance, swap symmetry,
    D mod 3 zero-padding (reading R5), sequence sharding (prefixed == unsharded).
"""
import glob
import json
import math
import os

import numpy as np
import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def rnd(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


def rand_problem(B, N, H, D, seed, n_prefix=0, scale=1.0):
    r = np.random.default_rng(seed)
    q = r.standard_normal((B, N, H, D)) * scale
    ks = [r.standard_normal((B, N + n_prefix, H, D)) * scale for _ in range(4)]
    dO = r.standard_normal((B, N, H, D))
    return q, ks[0], ks[1], ks[2], ks[3], dO


# ----------------------------------------------------------------------------------------------
# Independent dense reference built from Alg. 1: einsum -> masked softmax over the
# last two axes -> einsum back.  Used only as a pin.
# ----------------------------------------------------------------------------------------------
def window_mask(N, w1, w2):
    t = np.arange(N)[:, None]
    s = np.arange(N)[None, :]
    m1 = (s <= t) & (s > t - w1)          # [t, s]
    m2 = (s <= t) & (s > t - w2)          # [t, r]
    return m1[:, :, None] & m2[:, None, :]  # [t, s, r]


def det_logits_linalg(q, k, k2):
    """A^det via numpy.linalg.det on stacked 3x3 chunk matrices (Eq. logits)."""
    B, N, H, D = q.shape
    p = D // 3
    out = np.zeros((B, H, N, N, N))
    for l in range(p):
        sl = slice(3 * l, 3 * l + 3)
        qa = q[..., sl].transpose(0, 2, 1, 3)   # b n t 3
        ka = k[..., sl].transpose(0, 2, 1, 3)
        ca = k2[..., sl].transpose(0, 2, 1, 3)
        M = np.stack(np.broadcast_arrays(qa[:, :, :, None, None, :], ka[:, :, None, :, None, :],
                                         ca[:, :, None, None, :, :]), axis=-2)  # b n t s r 3 3
        out += np.linalg.det(M)
    return out


def alg1_numpy(q, k, v, k2, v2, w1, w2, det=False):
    B, N, H, D = q.shape
    if det:
        logits = det_logits_linalg(q, k, k2) / math.sqrt(D)
    else:
        logits = np.einsum("btnh,bsnh,brnh->bntsr", q, k, k2) / math.sqrt(D)
    mask = window_mask(N, w1, w2)
    logits = np.where(mask[None, None], logits, -np.inf)
    mx = logits.max(axis=(-1, -2), keepdims=True)
    e = np.exp(logits - mx)
    z = e.sum(axis=(-1, -2), keepdims=True)
    att = e / z
    out = np.einsum("bntsr,bsnh,brnh->btnh", att, v, v2)
    lse = (np.log(z) + mx)[..., 0, 0]
    return out, lse


def dense_torch(q, k, v, k2, v2, w1, w2, det=False):
    """Same model in torch float64 for autograd (dets via torch.linalg.det)."""
    B, N, H, D = q.shape
    if det:
        logits = 0
        for l in range(D // 3):
            sl = slice(3 * l, 3 * l + 3)
            qa, ka, ca = (x[..., sl].permute(0, 2, 1, 3) for x in (q, k, k2))
            M = torch.stack(torch.broadcast_tensors(qa[:, :, :, None, None, :], ka[:, :, None, :, None, :],
                                                    ca[:, :, None, None, :, :]), dim=-2)
            logits = logits + torch.linalg.det(M)
        logits = logits / math.sqrt(D)
    else:
        logits = torch.einsum("btnh,bsnh,brnh->bntsr", q, k, k2) / math.sqrt(D)
    mask = torch.from_numpy(window_mask(N, w1, w2))
    logits = logits.masked_fill(~mask[None, None], float("-inf"))
    att = torch.softmax(logits.flatten(-2), dim=-1).view_as(logits)
    return torch.einsum("bntsr,bsnh,brnh->btnh", att, v, v2)


# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(HERE, "golden", "*.json"))),
                         ids=lambda p: os.path.basename(p))
def test_golden(oracle_mod, path):
    g = json.load(open(path))
    shp = (g["B"], g["N"], g["H"], g["D"])
    arr = {n: np.array(g[n], dtype=np.float64).reshape(shp) for n in ("q", "k", "v", "k2", "v2")}
    o, lse = oracle_mod.forward(arr["q"], arr["k"], arr["v"], arr["k2"], arr["v2"], g["w1"], g["w2"],
                                det=g["variant"] == "det")
    np.testing.assert_allclose(lse.reshape(-1), np.array(g["lse"]), rtol=0, atol=1e-12)
    np.testing.assert_allclose(o.reshape(g["N"], g["D"]), np.array(g["o"]), rtol=0, atol=1e-12)


def test_det_row_swap_flips_sign(oracle_mod):
    e = np.eye(3).reshape(3, 1, 1, 1, 3)
    _, l1 = oracle_mod.forward(e[0], e[1], e[1], e[2], e[2], 1, 1, det=True)
    _, l2 = oracle_mod.forward(e[0], e[2], e[2], e[1], e[1], 1, 1, det=True)
    assert abs(l1.item() - 1 / math.sqrt(3)) < 1e-15 and abs(l2.item() + 1 / math.sqrt(3)) < 1e-15


@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("N,D,w1,w2", [(7, 6, 7, 7), (9, 6, 4, 3), (10, 5, 3, 6), (6, 3, 1, 1), (8, 7, 20, 2)])
def test_alg1_einsum(oracle_mod, N, D, w1, w2, det):
    """Alg. 1 literally, causal (w=N) and windowed; w > N clamps."""
    q, k, v, k2, v2, _ = rand_problem(2, N, 2, D, seed=N * 100 + D)
    o, lse = oracle_mod.forward(q, k, v, k2, v2, w1, w2, det=det)
    o_ref, lse_ref = alg1_numpy(q, k, v, k2, v2, w1, w2, det=det)
    np.testing.assert_allclose(o, o_ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(lse, lse_ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("w1,w2", [(5, 3), (16, 8), (3, 16)])
def test_collapse_to_dot_attention(oracle_mod, w1, w2):
    """K'=1, V'=1 -> sliding-window dot-product attention, computed by torch SDPA;
    lse shifts by ln(min(i+1, w2)) (reading R19)."""
    B, N, H, D = 2, 24, 3, 8
    q, k, v, _, _, _ = rand_problem(B, N, H, D, seed=7)
    ones = np.ones_like(k)
    o, lse = oracle_mod.forward(q, k, v, ones, ones, w1, w2)
    tq, tk, tv = (torch.from_numpy(x).permute(0, 2, 1, 3) for x in (q, k, v))
    i = torch.arange(N)[:, None]
    j = torch.arange(N)[None, :]
    mask = (j <= i) & (j > i - w1)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask)
    np.testing.assert_allclose(o, ref.permute(0, 2, 1, 3).numpy(), rtol=0, atol=1e-12)
    sc = (tq @ tk.transpose(-1, -2)) / math.sqrt(D)
    lse_dot = torch.logsumexp(sc.masked_fill(~mask, float("-inf")), dim=-1).numpy()
    shift = np.log(np.minimum(np.arange(N) + 1, w2))
    np.testing.assert_allclose(lse, lse_dot + shift, rtol=0, atol=1e-12)


@pytest.mark.parametrize("det", [False, True])
def test_convex_combination(oracle_mod, det):
    """V = V' = 1 -> O = 1: the softmax over each (j,k) window sums to 1 (Eq. softmax)."""
    q, k, _, k2, _, _ = rand_problem(1, 40, 2, 9, seed=3, scale=2.0)
    ones = np.ones_like(k)
    o, _ = oracle_mod.forward(q, k, ones, k2, ones, 13, 5, det=det)
    np.testing.assert_allclose(o, 1.0, rtol=0, atol=1e-13)


def random_so3(rng):
    a = rng.standard_normal((3, 3))
    qm, r = np.linalg.qr(a)
    qm = qm * np.sign(np.diag(r))
    if np.linalg.det(qm) < 0:
        qm[:, 0] = -qm[:, 0]
    return qm


def test_det_rotation_invariance(oracle_mod):
    """det logits are invariant under a common SO(3) rotation of every 3-chunk of q, k, k'
    (reading R7); the trilinear form is not."""
    rng = np.random.default_rng(11)
    B, N, H, D = 1, 20, 2, 8     # two chunks + 2 trailing dims (left unrotated)
    q, k, v, k2, v2, _ = rand_problem(B, N, H, D, seed=5)
    Rs = [random_so3(rng) for _ in range(D // 3)]

    def rot(x):
        y = x.copy()
        for l, R in enumerate(Rs):
            y[..., 3 * l:3 * l + 3] = x[..., 3 * l:3 * l + 3] @ R.T
        return y

    o1, l1 = oracle_mod.forward(q, k, v, k2, v2, 7, 4, det=True)
    o2, l2 = oracle_mod.forward(rot(q), rot(k), v, rot(k2), v2, 7, 4, det=True)
    np.testing.assert_allclose(l2, l1, rtol=0, atol=1e-11)
    np.testing.assert_allclose(o2, o1, rtol=0, atol=1e-11)
    _, t1 = oracle_mod.forward(q, k, v, k2, v2, 7, 4, det=False)
    _, t2 = oracle_mod.forward(rot(q), rot(k), v, rot(k2), v2, 7, 4, det=False)
    assert np.abs(t2 - t1).max() > 1e-3


def test_det_mod3_equals_zero_pad(oracle_mod):
    """D=8: trailing D mod 3 = 2 dims do not enter the logits == zero-padding to D=9 with the
    scale held at 1/sqrt(8) (reading R5); compare via unscaled logits ratio."""
    q, k, v, k2, v2, dO = rand_problem(1, 12, 1, 8, seed=9)
    o8, l8 = oracle_mod.forward(q, k, v, k2, v2, 5, 3, det=True)
    # Zero the trailing dims of q: must not change anything (they never enter the logits).
    qz = q.copy(); qz[..., 6:] = 0
    kz = k.copy(); kz[..., 6:] = 0
    o8z, l8z = oracle_mod.forward(qz, kz, v, k2, v2, 5, 3, det=True)
    np.testing.assert_array_equal(l8, l8z)
    np.testing.assert_array_equal(o8, o8z)
    dq, dk, dv, dk2, dv2 = oracle_mod.backward(q, k, v, k2, v2, dO, 5, 3, det=True)
    for g in (dq, dk, dk2):
        assert np.all(g[..., 6:] == 0)


@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("N,D,w1,w2", [(9, 6, 4, 3), (7, 4, 7, 2), (8, 7, 3, 5)])
def test_backward_autograd(oracle_mod, N, D, w1, w2, det):
    """All five gradients equal torch autograd of the dense Alg. 1 model (float64)."""
    if det and D < 3:
        pytest.skip()
    q, k, v, k2, v2, dO = rand_problem(2, N, 2, D, seed=N + D + 17)
    ts = [torch.from_numpy(x).requires_grad_(True) for x in (q, k, v, k2, v2)]
    out = dense_torch(*ts, w1, w2, det=det)
    out.backward(torch.from_numpy(dO))
    ref = [t.grad.numpy() for t in ts]   # dq, dk, dv, dk2, dv2
    got = oracle_mod.backward(q, k, v, k2, v2, dO, w1, w2, det=det)
    for n, gi, ri in zip(("dq", "dk", "dv", "dk2", "dv2"), got, ref):
        np.testing.assert_allclose(gi, ri, rtol=0, atol=1e-11, err_msg=n)


@pytest.mark.parametrize("det", [False, True])
def test_backward_finite_differences(oracle_mod, det):
    """Central differences of L = <dO, O>, h = 1e-4, normwise rel err <= 1e-6 (north star,
    reading R21)."""
    q, k, v, k2, v2, dO = rand_problem(1, 6, 1, 6, seed=23)
    w1, w2 = 4, 3
    grads = oracle_mod.backward(q, k, v, k2, v2, dO, w1, w2, det=det)
    base = [q, k, v, k2, v2]
    h = 1e-4
    for t in range(5):
        num = np.zeros_like(base[t])
        it = np.nditer(base[t], flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            args_p = [x.copy() for x in base]
            args_m = [x.copy() for x in base]
            args_p[t][idx] += h
            args_m[t][idx] -= h
            op, _ = oracle_mod.forward(*args_p, w1, w2, det=det)
            om, _ = oracle_mod.forward(*args_m, w1, w2, det=det)
            num[idx] = (np.sum(op * dO) - np.sum(om * dO)) / (2 * h)
        an = grads[t]
        rel = np.abs(num - an).max() / np.abs(an).max()
        assert rel <= 1e-6, (t, rel)


def test_single_position_closed_form(oracle_mod):
    """n=1: S=1 so O = v0 o v'0, dQ=dK=dK'=0, dV = dO o v'0, dV' = dO o v0."""
    q, k, v, k2, v2, dO = rand_problem(2, 1, 3, 5, seed=31)
    for det in (False, True):
        o, lse = oracle_mod.forward(q, k, v, k2, v2, 4, 4, det=det)
        np.testing.assert_allclose(o, v * v2, rtol=0, atol=1e-15)
        dq, dk, dv, dk2, dv2 = oracle_mod.backward(q, k, v, k2, v2, dO, 4, 4, det=det)
        for g in (dq, dk, dk2):
            np.testing.assert_allclose(g, 0, atol=1e-15)
        np.testing.assert_allclose(dv, dO * v2, atol=1e-15)
        np.testing.assert_allclose(dv2, dO * v, atol=1e-15)


def test_zero_cotangent(oracle_mod):
    q, k, v, k2, v2, dO = rand_problem(1, 10, 2, 4, seed=37)
    for g in oracle_mod.backward(q, k, v, k2, v2, np.zeros_like(dO), 4, 3):
        assert np.all(g == 0)


def test_swap_symmetry(oracle_mod):
    """(K,V,w1) <-> (K',V',w2) leaves the trilinear operator unchanged and swaps the gradients;
    for the determinant form the swap negates the logits, undone by q -> -q (A is linear in q)."""
    q, k, v, k2, v2, dO = rand_problem(2, 15, 2, 6, seed=41)
    o1, l1 = oracle_mod.forward(q, k, v, k2, v2, 6, 3)
    o2, l2 = oracle_mod.forward(q, k2, v2, k, v, 3, 6)
    np.testing.assert_allclose(o2, o1, atol=1e-13)
    np.testing.assert_allclose(l2, l1, atol=1e-13)
    g1 = oracle_mod.backward(q, k, v, k2, v2, dO, 6, 3)
    g2 = oracle_mod.backward(q, k2, v2, k, v, dO, 3, 6)
    for a, b in zip(g1, (g2[0], g2[3], g2[4], g2[1], g2[2])):
        np.testing.assert_allclose(a, b, atol=1e-12)
    od1, ld1 = oracle_mod.forward(q, k, v, k2, v2, 6, 3, det=True)
    od2, ld2 = oracle_mod.forward(-q, k2, v2, k, v, 3, 6, det=True)
    np.testing.assert_allclose(od2, od1, atol=1e-13)
    np.testing.assert_allclose(ld2, ld1, atol=1e-13)


@pytest.mark.parametrize("det", [False, True])
def test_sequence_sharding(oracle_mod, det):
    """Prefixed shards (n_prefix = max(w1,w2)-1 halo rows) reproduce the unsharded oracle:
    O and lse exactly, and the key-side gradients once halo partials are added back to the
    owning shard (DESIGN.md sequence-sharded mode)."""
    B, N, H, D, w1, w2, G = 1, 48, 2, 6, 7, 3, 4
    q, k, v, k2, v2, dO = rand_problem(B, N, H, D, seed=43)
    o, lse = oracle_mod.forward(q, k, v, k2, v2, w1, w2, det=det)
    full = oracle_mod.backward(q, k, v, k2, v2, dO, w1, w2, det=det)
    npf = max(w1, w2) - 1
    L = N // G
    acc = [np.zeros_like(x) for x in (k, v, k2, v2)]
    for r in range(G):
        a = r * L
        p = min(npf, a)
        sl_k = slice(a - p, a + L)
        sl_q = slice(a, a + L)
        ok, lk = oracle_mod.forward(q[:, sl_q], k[:, sl_k], v[:, sl_k], k2[:, sl_k], v2[:, sl_k],
                                    w1, w2, det=det, n_prefix=p)
        np.testing.assert_array_equal(ok, o[:, sl_q])
        np.testing.assert_array_equal(lk, lse[:, :, sl_q])
        g = oracle_mod.backward(q[:, sl_q], k[:, sl_k], v[:, sl_k], k2[:, sl_k], v2[:, sl_k],
                                dO[:, sl_q], w1, w2, det=det, n_prefix=p)
        np.testing.assert_array_equal(g[0], full[0][:, sl_q])
        for t in range(4):
            acc[t][:, sl_k] += g[t + 1]
    for t in range(4):
        np.testing.assert_allclose(acc[t], full[t + 1], rtol=0, atol=1e-14)


def test_sampled_rows(oracle_mod):
    q, k, v, k2, v2, _ = rand_problem(2, 30, 2, 4, seed=47)
    o, lse = oracle_mod.forward(q, k, v, k2, v2, 9, 4)
    rows = np.array([0, 5, 29, 30 + 7, 2 * 30 + 11, 3 * 30 + 29])
    os_, ls = oracle_mod.forward(q, k, v, k2, v2, 9, 4, rows=rows)
    flat_l = lse.reshape(-1)
    np.testing.assert_array_equal(ls.reshape(-1)[rows], flat_l[rows])
    assert np.isnan(ls.reshape(-1)[1])


@pytest.mark.parametrize("M", [3, 4, 5, 6])
def test_match3_theorem(oracle_mod, M):
    """Theorem 1 through the oracle's determinant logits: with the App. A embeddings
    (sa_testutil.match3_problem) the output at position i is >= 1/2 iff x_i + x_j1 + x_j2 = 0
    (mod M) for some causal j1, j2; the softmax splits weight between the beta matching pairs
    (value 1) and the blank pair (value 0), o = beta / (beta + 1)."""
    from sa_testutil import match3_problem, match3_truth
    rng = np.random.default_rng(M)
    D = 64
    c = 60.0 * math.sqrt(D)  # the kernel's fixed 1/sqrt(D) scale is absorbed into c
    for _ in range(40):
        xs = rng.integers(0, M, size=7)
        t = match3_problem(xs, M, c, D)
        N = t["q"].shape[1]
        o, _ = oracle_mod.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], N, N, det=True)
        got = o[0, 1:, 0, 0] >= 0.5 - 1e-3
        assert np.array_equal(got, match3_truth(xs, M)), (xs, o[0, 1:, 0, 0])


@pytest.mark.parametrize("H,Hk,det", [(4, 2, False), (4, 1, True), (6, 3, False)])
def test_gqa_against_autograd(oracle_mod, H, Hk, det):
    """Grouped-query oracle (forward_gqa / backward_gqa) against torch autograd of the dense
    Alg. 1 model whose key heads are expanded with repeat_interleave: autograd forms the
    group sums of the key-side gradients itself (S:110 head mapping h -> h // (H / H_kv))."""
    B, N, D, w1, w2 = 2, 10, 6, 5, 3
    rng = np.random.default_rng(H * 10 + Hk)
    q = rng.standard_normal((B, N, H, D))
    dO = rng.standard_normal((B, N, H, D))
    keys = [rng.standard_normal((B, N, Hk, D)) for _ in range(4)]
    o, _ = oracle_mod.forward_gqa(q, *keys, w1, w2, det=det)
    grads = oracle_mod.backward_gqa(q, *keys, dO, w1, w2, det=det)
    tq = torch.tensor(q, requires_grad=True)
    tk = [torch.tensor(x, requires_grad=True) for x in keys]
    exp = [t.repeat_interleave(H // Hk, dim=2) for t in tk]
    ro = dense_torch(tq, *exp, w1, w2, det=det)
    ro.backward(torch.tensor(dO))
    assert np.max(np.abs(o - ro.detach().numpy())) < 1e-12
    for g, t in zip(grads, [tq, *tk]):
        assert np.max(np.abs(g - t.grad.numpy())) < 1e-10


@pytest.mark.parametrize("w1,w2", [(5, 3), (3, 16)])
def test_bias_collapse_to_dot_attention(oracle_mod, w1, w2):
    """K2_BIAS / V2_BIAS on K' = V' = 0 with both biases 1: the shifted K', V' are all
    ones, so the output is sliding-window dot-product attention over (Q, K, V), computed by torch
    SDPA, and lse shifts by ln(min(i+1, w2)) (reading R19).  A bias added to the wrong operand (K or
    V instead of K' or V') fails this."""
    B, N, H, D = 1, 20, 2, 8
    q, k, v, _, _, _ = rand_problem(B, N, H, D, seed=11)
    zeros = np.zeros_like(k)
    o, lse = oracle_mod.forward_bias(q, k, v, zeros, zeros, w1, w2, 1.0, 1.0)
    tq, tk, tv = (torch.from_numpy(x).permute(0, 2, 1, 3) for x in (q, k, v))
    i = torch.arange(N)[:, None]
    j = torch.arange(N)[None, :]
    mask = (j <= i) & (j > i - w1)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask)
    np.testing.assert_allclose(o, ref.permute(0, 2, 1, 3).numpy(), rtol=0, atol=1e-12)
    sc = (tq @ tk.transpose(-1, -2)) / math.sqrt(D)
    lse_dot = torch.logsumexp(sc.masked_fill(~mask, float("-inf")), dim=-1).numpy()
    shift = np.log(np.minimum(np.arange(N) + 1, w2))
    np.testing.assert_allclose(lse, lse_dot + shift, rtol=0, atol=1e-12)


@pytest.mark.parametrize("H,Hk,det", [(2, 2, False), (4, 2, True)])
def test_bias_against_autograd(oracle_mod, H, Hk, det):
    """forward_bias / backward_bias against torch autograd of the dense Alg. 1 model fed K' + b and
    V' + b': autograd differentiates through the add, so its K'/V' gradients are with
    respect to the caller's unshifted tensors."""
    B, N, D, w1, w2 = 1, 9, 6, 4, 3
    b2k, b2v = 0.37, -1.25
    rng = np.random.default_rng(H * 7 + Hk)
    q = rng.standard_normal((B, N, H, D))
    dO = rng.standard_normal((B, N, H, D))
    keys = [rng.standard_normal((B, N, Hk, D)) for _ in range(4)]
    o, _ = oracle_mod.forward_bias(q, *keys, w1, w2, b2k, b2v, det=det)
    grads = oracle_mod.backward_bias(q, *keys, dO, w1, w2, b2k, b2v, det=det)
    tq = torch.tensor(q, requires_grad=True)
    tk = [torch.tensor(x, requires_grad=True) for x in keys]
    sh = [tk[0], tk[1], tk[2] + b2k, tk[3] + b2v]
    exp = [t.repeat_interleave(H // Hk, dim=2) for t in sh]
    ro = dense_torch(tq, *exp, w1, w2, det=det)
    ro.backward(torch.tensor(dO))
    assert np.max(np.abs(o - ro.detach().numpy())) < 1e-12
    for g, t in zip(grads, [tq, *tk]):
        assert np.max(np.abs(g - t.grad.numpy())) < 1e-10
