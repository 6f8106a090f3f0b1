"""Test-side helpers: run the oracle on the same seeded inputs the CUDA path sees, on a full
problem or on a window-exact slice of a large one (sampled checks at BASELINE sizes)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

TOL_F32 = 1e-4   # north star: fp32 path max abs error
TOL_BF16 = 2e-2  # north star: bf16-in / fp32-accumulate path max abs error


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
