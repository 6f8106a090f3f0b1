"""Test-side helpers: run the oracle on the same seeded inputs the CUDA path sees, on a full
problem or on a window-exact slice of a large one (sampled checks at BASELINE sizes)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

TOL_F32 = 1e-4   # north star: fp32 path max abs error
TOL_BF16 = 2e-2  # north star: bf16-in / fp32-accumulate path max abs error


def record_errors(errs: dict, tol: float, tag: str | None = None) -> None:
    """Print a parity test's worst max-abs error per tensor and append it to
    gpurun_out/parity_errors.jsonl (when that directory exists: the GPU runs)."""
    import json
    import os
    test = tag or os.environ.get("PYTEST_CURRENT_TEST", "?").split(" (")[0]
    rec = {"test": test, "tol": tol, "max_abs": {n: float(e) for n, e in errs.items()}}
    print("parity", json.dumps(rec))
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "parity_errors.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def maxabs(a, b) -> float:
    a = f64(a) if isinstance(a, torch.Tensor) else a
    b = f64(b) if isinstance(b, torch.Tensor) else b
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def oracle_slice(inp: dict, b: int, h: int, a: int, L: int, w1: int, w2: int, det: bool, bwd: bool):
    """Oracle on queries [a, a+L) of slice (b, h) with the key halo as prefix: exact for those
    query rows (o, lse, dq) and for key rows r in [a, a+L) whose every touching query
    (r .. r+w-1) lies inside [a, a+L) or past the sequence end."""
    N = inp["q"].shape[1]
    npf = min(a, max(w1, w2) - 1)
    sl_q, sl_k = slice(a, a + L), slice(a - npf, a + L)

    def cut(name, sl):
        return f64(inp[name][b:b + 1, sl, h:h + 1])

    q, dO = cut("q", sl_q), cut("dO", sl_q)
    k, v, k2, v2 = (cut(n, sl_k) for n in ("k", "v", "k2", "v2"))
    o, lse = oracle.forward(q, k, v, k2, v2, w1, w2, det=det, n_prefix=npf)
    res = {"o": o[0, :, 0], "lse": lse[0, 0], "npf": npf}
    if bwd:
        dq, dk, dv, dk2, dv2 = oracle.backward(q, k, v, k2, v2, dO, w1, w2, det=det, n_prefix=npf)
        res.update(dq=dq[0, :, 0])
        end = a + L
        for name, g, w in (("dk", dk, w1), ("dv", dv, w1), ("dk2", dk2, w2), ("dv2", dv2, w2)):
            # exact key rows (absolute positions): r in [a, a+L) with r + w - 1 < a+L or a+L == N
            hi = end if end == N else max(a, end - w + 1)
            res[name] = (a, hi, g[0, npf + 0:npf + (hi - a), 0])
    return res


# ---------------------------------------------------------------------------------------------
# Match3 (Theorem 1; construction App. A) through the determinant logits.
# ---------------------------------------------------------------------------------------------
def match3_problem(xs, M: int, c: float, D: int = 64):
    """Embeddings of App. A for a sequence whose position 0 is the blank token and positions
    1..n carry xs (values in [0, M)).  Chunk 0 (dims 0-2) and chunk 1 (dims 3-5) are the paper's
    q, k, k'; the 7th dimension of the paper's blank pair (a dot-product score the
    kernel does not have) becomes a third determinant chunk (dims 6-8): q = (c,0,0), and only
    the blank token has k = (0,1,0), k' = (0,0,1), so det = c for the blank pair and 0 for any
    pair with a regular token.  Values: 1 for regular tokens, 0 for the
    blank, so v_j1 o v'_j2 = 1 exactly for regular pairs.  Returns float64 [1, n+1, 1, D] arrays."""
    n = len(xs)
    N = n + 1
    th = np.zeros(N)
    th[1:] = 2 * np.pi * np.asarray(xs, dtype=np.float64) / M
    q = np.zeros((N, D))
    k = np.zeros((N, D))
    k2 = np.zeros((N, D))
    v = np.ones((N, D))
    v2 = np.ones((N, D))
    cs, sn = np.cos(th), np.sin(th)
    q[:, 0], q[:, 1], q[:, 3], q[:, 4], q[:, 6] = c * cs, c * sn, -c * sn, c * cs, c
    k[1:, 0], k[1:, 1], k[1:, 3], k[1:, 4] = sn[1:], cs[1:], -sn[1:], -cs[1:]
    k2[1:, 2], k2[1:, 5] = cs[1:], -sn[1:]
    k[0, 7], k2[0, 8] = 1.0, 1.0  # blank token (chunk 2)
    v[0] = 0.0
    v2[0] = 0.0
    return {n_: a[None, :, None, :] for n_, a in (("q", q), ("k", k), ("v", v), ("k2", k2), ("v2", v2))}


def match3_truth(xs, M: int):
    """Causal Match3: position i (1-based in the embedded sequence) matches iff there are
    j1, j2 in 1..i with x_i + x_j1 + x_j2 = 0 (mod M) (the kernel's windows are causal)."""
    out = []
    for i in range(len(xs)):
        hit = any((xs[i] + xs[a] + xs[b]) % M == 0 for a in range(i + 1) for b in range(i + 1))
        out.append(hit)
    return np.array(out)
