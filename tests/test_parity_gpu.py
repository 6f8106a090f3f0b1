"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle, element by element,
on the same seeded inputs.  Tolerances are the north star's: max abs 1e-4 for the fp32 path,
2e-2 for the bf16-input path (outputs written in fp32, SA_OUT_F32; reading R20)."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2507_02754_b200 as sa_pkg
from paper_2507_02754_b200 import binding as sa
from paper_2507_02754_b200.inputs import CONFIGS, make_inputs, seed_of
from sa_testutil import TOL_BF16, TOL_F32, f64, maxabs, oracle_slice, record_errors

pytestmark = pytest.mark.gpu
DEV = "cuda"


def run_cuda(inp, w1, w2, det, out_f32=True, n_prefix=0, force_simt=False, bwd=True):
    t = {n: x.to(DEV) for n, x in inp.items()}
    o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=det, out_f32=out_f32,
                        n_prefix=n_prefix, force_simt=force_simt)
    res = {"o": o, "lse": lse}
    if bwd:
        dq, dk, dv, dk2, dv2 = sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2,
                                           det=det, out_f32=out_f32, n_prefix=n_prefix, force_simt=force_simt)
        res.update(dq=dq, dk=dk, dv=dv, dk2=dk2, dv2=dv2)
    torch.cuda.synchronize()
    return res


def run_oracle(inp, w1, w2, det, n_prefix=0, bwd=True):
    a = {n: f64(x) for n, x in inp.items()}
    o, lse = oracle.forward(a["q"], a["k"], a["v"], a["k2"], a["v2"], w1, w2, det=det, n_prefix=n_prefix)
    res = {"o": o, "lse": lse}
    if bwd:
        g = oracle.backward(a["q"], a["k"], a["v"], a["k2"], a["v2"], a["dO"], w1, w2, det=det, n_prefix=n_prefix)
        res.update(zip(("dq", "dk", "dv", "dk2", "dv2"), g))
    return res


def assert_close(got, ref, tol, names=("o", "lse", "dq", "dk", "dv", "dk2", "dv2")):
    errs = {n: maxabs(got[n], ref[n]) for n in names if n in got}
    record_errors(errs, tol)
    bad = {n: e for n, e in errs.items() if not e <= tol}
    assert not bad, f"max abs errors {errs} exceed {tol}"
    return errs


def test_c1_fp32_full():
    """BASELINE config 1 (fp32, B=1 H=1 N=128 D=16 w1=32 w2=8), fwd+bwd, whole tensors."""
    c = CONFIGS["c1"]
    inp = make_inputs(c["B"], c["N"], c["H"], c["D"], seed_of("c1"), dtype="f32")
    got = run_cuda(inp, c["w1"], c["w2"], False)
    ref = run_oracle(inp, c["w1"], c["w2"], False)
    assert_close(got, ref, TOL_F32)


@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("B,N,H,D,w1,w2", [
    (1, 1, 1, 16, 4, 4),        # single position
    (2, 77, 3, 16, 9, 4),       # ragged N
    (1, 64, 2, 32, 100, 3),     # window longer than the sequence (clamps)
    (1, 96, 1, 48, 5, 17),      # w2 > w1
    (1, 130, 2, 128, 33, 8),    # D = 128
    (1, 50, 1, 7, 6, 6),        # D not a multiple of 3 or 32
])
def test_fp32_shapes(B, N, H, D, w1, w2, det):
    inp = make_inputs(B, N, H, D, seed=N + D, dtype="f32")
    got = run_cuda(inp, w1, w2, det)
    ref = run_oracle(inp, w1, w2, det)
    assert_close(got, ref, TOL_F32)


@pytest.mark.parametrize("force_simt", [False, True])
@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("B,N,H,D,w1,w2", [
    (1, 384, 2, 128, 64, 32),
    (1, 300, 1, 128, 128, 32),   # ragged tail, several tiles
    (2, 256, 1, 64, 48, 16),     # D = 64
    (1, 200, 1, 128, 40, 64),    # w2 = 64
    (1, 160, 1, 128, 16, 48),    # w2 > w1
    (1, 300, 2, 128, 128, 64),   # R = 64 rows per query (G = 2): the c5 / Table-1 (512, 64) tiling
    (2, 170, 1, 128, 96, 64),    # R = 64, ragged tail
    (1, 200, 2, 128, 32, 8),     # R = 8 (G = 16): the memory-bound small-window point of §8(d)
    (1, 96, 1, 64, 20, 4),       # R = 4
    (1, 70, 1, 128, 10, 2),      # R = 2 (G = 64)
    (1, 180, 2, 128, 24, 16),    # R = 16, D = 128 (G = 8: the band gather has G < R terms)
    (1, 150, 1, 128, 12, 5),     # w2 = 5 -> R = 8 with masked rows
    (1, 400, 1, 128, 128, 128),  # R = 128 (G = 1): Table 1's (128, 128) row, dK'/dV' ring in global memory
    (1, 300, 2, 64, 200, 128),   # R = 128, D = 64, ragged
    (1, 260, 1, 128, 128, 300),  # w2 > w1 = 128: swapped, R = 128
    (1, 1, 1, 128, 4, 4),        # N = 1: one query, one key
    (2, 150, 1, 128, 64, 1),     # w2 = 1 (R = 1, G = 128): forward generic epilogue; backward tiles of R = 2
    (1, 200, 1, 128, 96, 40),    # R = 40: forward G = 3; backward pads each query to 64 rows
    (1, 100, 2, 64, 24, 3),      # R = 3, D = 64: backward pads to 4 rows
    # window split: w2 > 32 runs as sub-windows of <= 32 K' rows
    (1, 300, 1, 128, 64, 96),    # 3 sub-windows of 32, forward and backward split
    (1, 300, 2, 128, 600, 72),   # w1 clamps to 300 (> 256): forward R = 72 unsplit, backward 32 + 32 + 8
    (1, 250, 1, 64, 100, 200),   # swapped: folded window 100 = 32 + 32 + 32 + 4, D = 64
])
def test_bf16_shapes(B, N, H, D, w1, w2, det, force_simt):
    inp = make_inputs(B, N, H, D, seed=7 * N + D, dtype="bf16")
    got = run_cuda(inp, w1, w2, det, force_simt=force_simt)
    ref = run_oracle(inp, w1, w2, det)
    assert_close(got, ref, TOL_BF16)


@pytest.mark.parametrize("det", [False, True])
def test_bf16_outputs_in_bf16(det):
    """Default output dtype (bf16) round-trips: compare against the oracle at the bf16 storage
    tolerance (|x| up to ~10 rounds by up to 2^-5; reading R20)."""
    inp = make_inputs(1, 256, 2, 128, seed=5, dtype="bf16")
    got = run_cuda(inp, 64, 32, det, out_f32=False)
    ref = run_oracle(inp, 64, 32, det)
    for n in ("o", "dq", "dk", "dv", "dk2", "dv2"):
        assert got[n].dtype == torch.bfloat16
        err = np.abs(f64(got[n]) - ref[n]) - 2.0 ** -8 * np.abs(ref[n])
        assert err.max() <= TOL_BF16, n


@pytest.mark.parametrize("win", [(40, 16), (96, 64)])  # (96, 64): window split with a halo prefix
@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("dtype,tol", [("f32", TOL_F32), ("bf16", TOL_BF16)])
def test_prefixed_mode(dtype, tol, det, win):
    """Sequence-sharded entry points: queries with a key halo as prefix, both variants."""
    (w1, w2) = win
    B, N, H, D, npf = 1, 160, 2, 64, max(w1, w2) - 1
    inp = make_inputs(B, N, H, D, seed=11, dtype=dtype, n_prefix=npf)
    got = run_cuda(inp, w1, w2, det, n_prefix=npf)
    ref = run_oracle(inp, w1, w2, det, n_prefix=npf)
    assert_close(got, ref, tol)


# Power-of-two rescalings that leave the logits and o unchanged (q a, k c, k2 b with abc = 1;
# v e, v2 f with ef = 1; dO g): exact in bf16 and float64, so the oracle's unscaled result fixes the
# expected values, while the fp16 MMA operands (q o k2, dO o v2; header INPUT RANGE) see large or
# small magnitudes.  Expected gradient scales: dq g/a, dk g/c, dk2 g/b, dv g f, dv2 g e.
INPUT_SCALES = {
    "large": dict(q=2.0 ** 4, k=2.0 ** -8, k2=2.0 ** 4, v=2.0 ** -3, v2=2.0 ** 3, dO=2.0 ** 3),
    "small": dict(q=2.0 ** -5, k=2.0 ** 10, k2=2.0 ** -5, v=2.0 ** 5, v2=2.0 ** -5, dO=2.0 ** -5),
}


@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("scale", sorted(INPUT_SCALES))
def test_input_scale(scale, det):
    """Input-range stress of the bf16 path (q o k2 up to ~2^8 x unit products, or down to 2^-10;
    dO o v2 likewise): every output, divided by its exact power-of-two scale, within the north-star
    tolerance of the oracle."""
    sc = INPUT_SCALES[scale]
    B, N, H, D, w1, w2 = 1, 256, 2, 128, 96, 32
    inp = make_inputs(B, N, H, D, seed=41, dtype="bf16")
    scaled = {n: (x.float() * sc[n]).to(torch.bfloat16) for n, x in inp.items()}
    for n in inp:  # powers of two: the rescaled bf16 values are exact
        assert torch.equal(scaled[n].float(), inp[n].float() * sc[n]), n
    got = run_cuda(scaled, w1, w2, det)
    ref = run_oracle(inp, w1, w2, det)
    g = sc["dO"]
    gscale = {"o": 1.0, "lse": 1.0, "dq": g / sc["q"], "dk": g / sc["k"], "dk2": g / sc["k2"],
              "dv": g * sc["v2"], "dv2": g * sc["v"]}
    unscaled = {n: got[n].double() / gscale[n] for n in gscale}
    for n in unscaled:
        assert torch.isfinite(got[n]).all(), n
    assert_close(unscaled, ref, TOL_BF16)


def test_tensor_core_path_selected():
    """bf16 inputs with D in {64,128} and a folded window <= 128 must run the tcgen05 kernels."""
    assert sa.fwd_path(4, 16, 8192, 128, 512, 32) == sa.SA_PATH_TCGEN05
    assert sa.fwd_path(2, 16, 16384, 128, 512, 32, det=True) == sa.SA_PATH_TCGEN05
    assert sa.fwd_path(1, 2, 256, 64, 16, 48) == sa.SA_PATH_TCGEN05
    assert sa.fwd_path(1, 2, 256, 128, 512, 32, dtype=torch.float32) == sa.SA_PATH_SIMT


def test_deterministic():
    inp = make_inputs(1, 300, 2, 128, seed=3, dtype="bf16")
    a = run_cuda(inp, 128, 32, False)
    b = run_cuda(inp, 128, 32, False)
    for n in a:
        assert torch.equal(a[n], b[n]), n


@pytest.mark.parametrize("B", [1, 3])
def test_host_step_matches_device_path(B):
    """The end-to-end host step (pipelined per batch element when B > 1) reproduces the device
    path: bitwise where the per-slice decomposition is the same (o, lse, dq, dk, dv); dk2/dv2 may
    differ in fp32 summation order because the per-CTA tile ranges of bwd_q depend on B."""
    N, H, D, w1, w2 = 256, 2, 128, 64, 32
    inp = make_inputs(B, N, H, D, seed=17, dtype="bf16")
    dev = run_cuda(inp, w1, w2, False)
    h_in = {n: x.pin_memory() for n, x in inp.items()}
    h_out = {n: torch.empty(dev[n].shape, dtype=dev[n].dtype).pin_memory() for n in dev}
    sa.host_step(h_in, h_out, w1, w2, out_f32=True)
    torch.cuda.synchronize()
    for n in dev:
        if n in ("dk2", "dv2"):
            assert torch.allclose(h_out[n], dev[n].cpu(), rtol=0, atol=1e-4), n
        else:
            assert torch.equal(h_out[n], dev[n].cpu()), n


# The memory-bound small-window point of SURVEY.md Sec. 8(d) (bench.py --sweep membound): windows 32 x 8
# at the c3 shape, run by the R = 8 kernels (pitched-row TMA staging, tensor-core row-group sums)
MEMBOUND = dict(B=4, H=16, N=8192, D=128, w1=32, w2=8, dtype="bf16", det=False, bwd=True)


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5", "membound"])
def test_baseline_config_sampled(cfg):
    """Full BASELINE sizes in the bench's launch configuration; the oracle checks 16 sampled
    (b, h, query-range) slices window-exactly (sa_testutil.oracle_slice).  Each slice spans
    L = w1 + 128 queries, so besides o, lse, dq (all L rows) and dk2/dv2 (L - w2 + 1 rows), 129
    interior key rows of dk/dv -- rows whose every touching query lies inside the slice -- are
    compared; the first and last slices also cover the sequence start and end."""
    c = CONFIGS[cfg] if cfg in CONFIGS else MEMBOUND
    inp = make_inputs(c["B"], c["N"], c["H"], c["D"], seed_of(cfg) if cfg in CONFIGS else 6000, dtype=c["dtype"],
                      device="cpu")
    got = run_cuda(inp, c["w1"], c["w2"], c["det"], bwd=c["bwd"])
    N, L = c["N"], c["w1"] + 128
    rng = np.random.default_rng(0)
    samples = [(0, 0, 0), (c["B"] - 1, c["H"] - 1, N - L)]
    while len(samples) < 16:
        samples.append((int(rng.integers(c["B"])), int(rng.integers(c["H"])), int(rng.integers(1, N - L))))
    worst = {}
    n_interior = 0
    for b, h, a in samples:
        ref = oracle_slice(inp, b, h, a, L, c["w1"], c["w2"], c["det"], c["bwd"])
        errs = {"o": maxabs(got["o"][b, a:a + L, h], ref["o"]),
                "lse": maxabs(got["lse"][b, h, a:a + L], ref["lse"])}
        if c["bwd"]:
            errs["dq"] = maxabs(got["dq"][b, a:a + L, h], ref["dq"])
            for n in ("dk", "dv", "dk2", "dv2"):
                lo, hi, r = ref[n]
                assert hi - lo >= (L - c["w1"] + 1 if n in ("dk", "dv") else L - c["w2"] + 1) or a + L == N
                errs[n] = maxabs(got[n][b, lo:hi, h], r)
            n_interior += ref["dk"][1] - ref["dk"][0]
        for n, e in errs.items():
            worst[n] = max(worst.get(n, 0.0), e)
        assert all(e <= TOL_BF16 for e in errs.values()), (cfg, b, h, a, errs)
    record_errors(worst, TOL_BF16, tag=f"{cfg} sampled x{len(samples)}")
    if c["bwd"]:
        assert n_interior >= 16 * 129


@pytest.mark.parametrize("det", [False, True])
def test_sequence_sharded_cuda_simulated(det):
    """The sequence-sharded composition (parallel.py) with the CUDA kernels, ranks simulated in one
    process: each shard runs the prefixed entry points with a max(w1,w2)-1 row halo, halo-row
    gradients are added back to their owner; the result matches the unsharded CUDA run."""
    B, N, H, D, w1, w2, world = 1, 512, 2, 128, 96, 32, 4
    inp = make_inputs(B, N, H, D, seed=21, dtype="bf16")
    full = run_cuda(inp, w1, w2, det)
    L, nh = N // world, max(w1, w2) - 1
    key_acc = {n: torch.zeros_like(full[n]) for n in ("dk", "dv", "dk2", "dv2")}
    for r in range(world):
        lo = r * L
        npf = min(nh, lo)
        sl_q, sl_k = slice(lo, lo + L), slice(lo - npf, lo + L)
        shard = {n: (x[:, sl_k] if n in ("k", "v", "k2", "v2") else x[:, sl_q]).contiguous() for n, x in inp.items()}
        got = run_cuda(shard, w1, w2, det, n_prefix=npf)
        assert maxabs(got["o"], full["o"][:, sl_q]) <= 1e-5
        assert maxabs(got["lse"], full["lse"][:, :, sl_q]) <= 1e-5
        assert maxabs(got["dq"], full["dq"][:, sl_q]) <= 1e-4
        for n in key_acc:
            key_acc[n][:, sl_k] += got[n]
    for n in key_acc:
        assert maxabs(key_acc[n], full[n]) <= 1e-4, n


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_autograd_wrapper(dtype):
    """torch.autograd through simplicial_attention reproduces the direct forward/backward calls
    (and hence the oracle): o and all five gradients, bitwise."""
    B, N, H, D, w1, w2 = 1, 192, 2, 64, 48, 16
    inp = make_inputs(B, N, H, D, seed=29, dtype=dtype)
    t = {n: x.cuda() for n, x in inp.items()}
    leaves = {n: t[n].clone().requires_grad_(True) for n in ("q", "k", "v", "k2", "v2")}
    o = sa_pkg.simplicial_attention(leaves["q"], leaves["k"], leaves["v"], leaves["k2"], leaves["v2"], w1, w2)
    o.backward(t["dO"])
    o_ref, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2)
    grads = sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o_ref, lse, t["dO"], w1, w2)
    assert torch.equal(o, o_ref)
    for n, g in zip(("q", "k", "v", "k2", "v2"), grads):
        assert torch.equal(leaves[n].grad, g), n


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_match3_det_kernel(dtype):
    """Theorem 1's Match3 construction (App. A) evaluated by the CUDA determinant path: bf16 inputs
    on the tcgen05 kernel (M = 4: every sin/cos is exact in bf16, so the match score is exactly c)
    and fp32 inputs on the exact path (M = 6)."""
    from sa_testutil import match3_problem, match3_truth
    M = 4 if dtype == "bf16" else 6
    D = 64
    c = 40.0 * math.sqrt(D)
    rng = np.random.default_rng(7)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    for _ in range(8):
        xs = rng.integers(0, M, size=31)
        t = {n: torch.from_numpy(a).to(tdt).cuda() for n, a in match3_problem(xs, M, c, D).items()}
        N = t["q"].shape[1]
        o, _ = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], N, N, det=True, out_f32=True)
        if dtype == "bf16":
            assert sa.fwd_path(1, 1, N, D, N, N, det=True) == sa.SA_PATH_TCGEN05
        got = o[0, 1:, 0, 0].double().cpu().numpy() >= 0.5 - 1e-3
        assert np.array_equal(got, match3_truth(xs, M)), xs


@pytest.mark.parametrize("dtype,tol", [("bf16", TOL_BF16), ("f32", TOL_F32)])
@pytest.mark.parametrize("H,Hk,D,w1,w2,det", [
    (4, 2, 128, 96, 32, False),   # tcgen05 path, ratio 2
    (8, 1, 64, 64, 16, True),     # all query heads share one key head (det)
    (4, 4, 128, 64, 32, False),   # H_kv == H: the ordinary path through the GQA entry points
    (4, 2, 128, 80, 70, True),    # window split with grouped keys (sub-windows 32 + 32 + 6), det
])
def test_gqa(dtype, tol, H, Hk, D, w1, w2, det):
    """Grouped-query entry points against the grouped-query oracle (expand + group sums)."""
    B, N = 2, 200
    g = torch.Generator().manual_seed(H * 100 + Hk)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q, dO = (torch.randn(B, N, H, D, generator=g).to(dt) for _ in range(2))
    keys = [torch.randn(B, N, Hk, D, generator=g).to(dt) for _ in range(4)]
    t = [x.to(DEV) for x in (q, *keys, dO)]
    o, lse = sa.forward(*t[:5], w1, w2, det=det, out_f32=True)
    grads = sa.backward(*t[:5], o, lse, t[5], w1, w2, det=det, out_f32=True)
    torch.cuda.synchronize()
    a = [f64(x) for x in (q, *keys, dO)]
    ro, rl = oracle.forward_gqa(*a[:5], w1, w2, det=det)
    rg = oracle.backward_gqa(*a[:5], a[5], w1, w2, det=det)
    got = dict(zip(("o", "lse", "dq", "dk", "dv", "dk2", "dv2"), (o, lse, *grads)))
    ref = dict(zip(("o", "lse", "dq", "dk", "dv", "dk2", "dv2"), (ro, rl, *rg)))
    assert_close(got, ref, tol)
    if Hk < H:  # bf16 outputs: the reduction writes the output dtype
        o16, lse16 = sa.forward(*t[:5], w1, w2, det=det)
        g16 = sa.backward(*t[:5], o16, lse16, t[5], w1, w2, det=det)
        assert all(x.dtype == (torch.bfloat16 if dtype == "bf16" else torch.float32) for x in g16)
        assert maxabs(g16[1], rg[1]) <= 4 * TOL_BF16


@pytest.mark.parametrize("dtype,tol", [("bf16", TOL_BF16), ("f32", TOL_F32)])
@pytest.mark.parametrize("H,Hk,D,w1,w2,det", [
    (2, 2, 128, 96, 32, False),   # multi-head, tcgen05 path
    (4, 2, 64, 64, 16, True),     # grouped-query, determinant
])
def test_bias(dtype, tol, H, Hk, D, w1, w2, det):
    """K2_BIAS / V2_BIAS entry points against the oracle's forward_bias / backward_bias
    (float64 add of the scalars, then the method); also through the autograd wrapper."""
    B, N = 2, 160
    b2k, b2v = 0.37, -1.25
    g = torch.Generator().manual_seed(H * 10 + D)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q, dO = (torch.randn(B, N, H, D, generator=g).to(dt) for _ in range(2))
    keys = [torch.randn(B, N, Hk, D, generator=g).to(dt) for _ in range(4)]
    t = [x.to(DEV) for x in (q, *keys, dO)]
    o, lse = sa.forward(*t[:5], w1, w2, det=det, out_f32=True, k2_bias=b2k, v2_bias=b2v)
    grads = sa.backward(*t[:5], o, lse, t[5], w1, w2, det=det, out_f32=True, k2_bias=b2k, v2_bias=b2v)
    torch.cuda.synchronize()
    a = [f64(x) for x in (q, *keys, dO)]
    if dtype == "bf16":
        # the paper casts k2 + K2_BIAS to the GEMM dtype bf16; the bias entry points also
        # round v2 + V2_BIAS to bf16 (reading R14): the oracle gets the same rounded shifted rows
        # (fp32 add, round to nearest even), passed with zero bias
        sk2, sv2 = ((x.float() + b).to(torch.bfloat16) for x, b in ((keys[2], b2k), (keys[3], b2v)))
        ab, bk, bv = [*a[:3], f64(sk2), f64(sv2)], 0.0, 0.0
    else:
        ab, bk, bv = a[:5], b2k, b2v
    ro, rl = oracle.forward_bias(*ab, w1, w2, bk, bv, det=det)
    rg = oracle.backward_bias(*ab, a[5], w1, w2, bk, bv, det=det)
    got = dict(zip(("o", "lse", "dq", "dk", "dv", "dk2", "dv2"), (o, lse, *grads)))
    ref = dict(zip(("o", "lse", "dq", "dk", "dv", "dk2", "dv2"), (ro, rl, *rg)))
    assert_close(got, ref, tol)
    # the caller's k2 / v2 are untouched (the biased copies live in the workspace)
    assert torch.equal(t[3].cpu(), keys[2]) and torch.equal(t[4].cpu(), keys[3])
    if Hk == H:
        leaves = [x.clone().requires_grad_(True) for x in t[:5]]
        oa = sa_pkg.simplicial_attention(*leaves, w1, w2, det=det, k2_bias=b2k, v2_bias=b2v)
        oa.backward(t[5])
        o_d, lse_d = sa.forward(*t[:5], w1, w2, det=det, k2_bias=b2k, v2_bias=b2v)
        g_d = sa.backward(*t[:5], o_d, lse_d, t[5], w1, w2, det=det, k2_bias=b2k, v2_bias=b2v)
        assert torch.equal(oa, o_d)
        for lf, gd in zip(leaves, g_d):
            assert torch.equal(lf.grad, gd)


@pytest.mark.parametrize("det", [False, True])
def test_r128_backward_on_tcgen05(det):
    """w2 = 128 (Table 1's (128, 128) row) runs the tcgen05 backward, not the CUDA-core path."""
    assert sa.bwd_path(1, 16, 8192, 128, 128, 128, det=det) == sa.SA_PATH_TCGEN05
    assert sa.fwd_path(1, 16, 8192, 128, 128, 128, det=det) == sa.SA_PATH_TCGEN05


@pytest.mark.parametrize("det", [False, True])
def test_unsplit_tiling(det):
    """SA_NO_WSPLIT=1 (read once per process) keeps the single R = 64 / 128 tilings of the folded
    window instead of the window split: run them in a child process against the oracle."""
    import json
    import os
    import subprocess
    import sys
    code = f"""
import json, sys
sys.path[:0] = {[os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__))]!r}
from sa_testutil import maxabs
from test_parity_gpu import run_cuda, run_oracle
from paper_2507_02754_b200.inputs import make_inputs
out = {{}}
for (N, w1, w2) in ((300, 128, 64), (200, 64, 128)):
    inp = make_inputs(1, N, 2, 128, seed=N, dtype="bf16")
    got = run_cuda(inp, w1, w2, {det})
    ref = run_oracle(inp, w1, w2, {det})
    out[f"{{w1}}x{{w2}}"] = {{n: maxabs(got[n], ref[n]) for n in got}}
print(json.dumps(out))
"""
    env = dict(os.environ, SA_NO_WSPLIT="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for shape, errs in res.items():
        record_errors(errs, TOL_BF16, tag=f"test_unsplit_tiling[{det}]::{shape}")
        assert all(e <= TOL_BF16 for e in errs.values()), (shape, errs)
