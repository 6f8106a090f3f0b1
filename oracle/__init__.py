"""float64 CPU oracle for sliding-window 2-simplicial attention (Sec. 4-7).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  It shares no code with ``paper_2507_02754_b200`` and neither imports
the other.  The arithmetic lives in ``oracle.c`` (plain C, float64, OpenMP);
this file only marshals numpy arrays through ctypes.

Functions
---------
forward(q, k, v, k2, v2, w1, w2, det=False, n_prefix=0) -> (o, lse)
    Eq. 3d-attention / Eq. logits, Eq. softmax, Eq. attenval (P:230-245,
    P:291-301), windows j in (i-w1, i], k in (i-w2, i].
backward(q, k, v, k2, v2, dO, w1, w2, det=False, n_prefix=0) -> (dq, dk, dv, dk2, dv2)
    Corrected Sec. 7 equations, see DESIGN.md readings.

forward_gqa(q, k, v, k2, v2, w1, w2, det=False) / backward_gqa(...)
    Grouped-query attention (GQA ratio 64 in the paper's
    model; head mapping S:110): key-side tensors carry H_kv heads and
    query head h reads key head h // (H / H_kv).  Written as its definition: the
    key heads are repeated to H and the plain oracle runs; each key-side gradient
    is the sum of the gradients of the query heads that share it (chain rule).

forward_bias(q, k, v, k2, v2, w1, w2, k2_bias, v2_bias, det=False) / backward_bias(...)
    K2_BIAS / V2_BIAS of the paper's kernel listing: after loading,
    ``k2t_tile += K2_BIAS; v2_tile += V2_BIAS``, i.e. the method runs on
    K' + b and V' + b'.  Written as that: the scalars are added in float64 and the
    (grouped-query) oracle runs on the shifted tensors; the gradients with respect to
    K' and V' are those with respect to the shifted tensors (d(x + b)/dx = 1).

All arrays are float64 numpy arrays; q/dO are [B, N, H, D], key-side tensors
are [B, n_prefix+N, H, D] (query row i sits at key position n_prefix+i).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (-O2 -fopenmp).  Plain C, no GPU code."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.sa_oracle_fwd.argtypes = [P] * 7 + [I] * 7 + [ctypes.c_int, P, I]
        lib.sa_oracle_fwd.restype = None
        lib.sa_oracle_bwd.argtypes = [P] * 11 + [I] * 7 + [ctypes.c_int]
        lib.sa_oracle_bwd.restype = None
        lib.sa_oracle_threads.restype = ctypes.c_int
        lib.sa_oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _f64(x) -> np.ndarray:
    if hasattr(x, "detach"):  # torch tensor -> numpy without importing torch here
        x = x.detach().cpu().double().numpy()
    return np.ascontiguousarray(x, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _shapes(q, k, n_prefix):
    B, N, H, D = q.shape
    assert k.shape == (B, n_prefix + N, H, D), (k.shape, q.shape, n_prefix)
    return B, N, H, D


def set_threads(n: int) -> None:
    _load().sa_oracle_set_threads(int(n))


def threads_used() -> int:
    """OpenMP threads the last oracle call ran with."""
    return int(_load().sa_oracle_threads())


def forward(q, k, v, k2, v2, w1, w2, det=False, n_prefix=0, rows=None):
    """Returns (o [B,N,H,D], lse [B,H,N]) in float64.  ``rows`` (optional) restricts the
    computation to flat query indices (b*H+h)*N+i; other entries are NaN."""
    q, k, v, k2, v2 = map(_f64, (q, k, v, k2, v2))
    B, N, H, D = _shapes(q, k, n_prefix)
    for t in (v, k2, v2):
        assert t.shape == k.shape
    o = np.full((B, N, H, D), np.nan)
    lse = np.full((B, H, N), np.nan)
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        rp, nr = _ptr(rows), rows.size
    else:
        rp, nr = None, 0
    _load().sa_oracle_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(o), _ptr(lse),
                          B, H, N, D, int(w1), int(w2), int(n_prefix), int(bool(det)), rp, nr)
    return o, lse


def backward(q, k, v, k2, v2, dO, w1, w2, det=False, n_prefix=0):
    """Returns (dq, dk, dv, dk2, dv2) in float64 (key-side grads over all n_prefix+N rows)."""
    q, k, v, k2, v2, dO = map(_f64, (q, k, v, k2, v2, dO))
    B, N, H, D = _shapes(q, k, n_prefix)
    assert dO.shape == q.shape
    dq = np.empty_like(q)
    dk, dv, dk2, dv2 = (np.empty_like(k) for _ in range(4))
    _load().sa_oracle_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(dO),
                          _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dk2), _ptr(dv2),
                          B, H, N, D, int(w1), int(w2), int(n_prefix), int(bool(det)))
    return dq, dk, dv, dk2, dv2


def _repeat_heads(t: np.ndarray, r: int) -> np.ndarray:
    return np.ascontiguousarray(np.repeat(t, r, axis=2))  # [kv0]*r, [kv1]*r, ...: head h -> h // r


def forward_gqa(q, k, v, k2, v2, w1, w2, det=False):
    q, k, v, k2, v2 = map(_f64, (q, k, v, k2, v2))
    H, Hk = q.shape[2], k.shape[2]
    assert H % Hk == 0
    r = H // Hk
    return forward(q, *(_repeat_heads(t, r) for t in (k, v, k2, v2)), w1, w2, det=det)


def backward_gqa(q, k, v, k2, v2, dO, w1, w2, det=False):
    q, k, v, k2, v2, dO = map(_f64, (q, k, v, k2, v2, dO))
    B, NK, Hk, D = k.shape
    r = q.shape[2] // Hk
    dq, *gk = backward(q, *(_repeat_heads(t, r) for t in (k, v, k2, v2)), dO, w1, w2, det=det)
    return (dq, *(g.reshape(B, NK, Hk, r, D).sum(axis=3) for g in gk))


def forward_bias(q, k, v, k2, v2, w1, w2, k2_bias, v2_bias, det=False):
    k2, v2 = _f64(k2), _f64(v2)
    return forward_gqa(q, k, v, k2 + float(k2_bias), v2 + float(v2_bias), w1, w2, det=det)


def backward_bias(q, k, v, k2, v2, dO, w1, w2, k2_bias, v2_bias, det=False):
    k2, v2 = _f64(k2), _f64(v2)
    return backward_gqa(q, k, v, k2 + float(k2_bias), v2 + float(v2_bias), dO, w1, w2, det=det)
