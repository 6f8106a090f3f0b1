"""ctypes binding of libsimplicial.so -- argument marshalling only.

Every function here allocates outputs with torch on the inputs' CUDA device, passes raw
pointers and the current CUDA stream to the C ABI (include/simplicial_attn.h) and checks
the returned status.  No arithmetic of the method happens in Python.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _build

SA_VARIANT_DET = 1 << 0
SA_IN_F32 = 1 << 1
SA_OUT_F32 = 1 << 2
SA_FORCE_SIMT = 1 << 3
SA_PATH_SIMT = 1
SA_PATH_TCGEN05 = 2

_STATUS = {0: "SA_OK", 1: "SA_ERR_INVALID_ARG", 2: "SA_ERR_UNSUPPORTED", 3: "SA_ERR_WORKSPACE",
           4: "SA_ERR_CUDA"}
EXPORTS = (
    "simplicial_attn_fwd", "simplicial_attn_fwd_prefixed", "simplicial_attn_fwd_workspace_bytes",
    "simplicial_attn_fwd_workspace_bytes_prefixed", "simplicial_attn_bwd_workspace_bytes",
    "simplicial_attn_bwd_workspace_bytes_prefixed",
    "simplicial_attn_bwd", "simplicial_attn_bwd_prefixed", "simplicial_attn_host_step_scratch_bytes",
    "simplicial_attn_host_step", "simplicial_attn_fwd_path", "simplicial_attn_bwd_path",
    "simplicial_attn_launch_count", "simplicial_attn_status_string", "simplicial_attn_version",
    "simplicial_attn_profile_enable", "simplicial_attn_profile_read",
    "simplicial_attn_fwd_gqa_workspace_bytes", "simplicial_attn_fwd_gqa",
    "simplicial_attn_bwd_gqa_workspace_bytes", "simplicial_attn_bwd_gqa",
    "simplicial_attn_fwd_bias_workspace_bytes", "simplicial_attn_fwd_bias",
    "simplicial_attn_bwd_bias_workspace_bytes", "simplicial_attn_bwd_bias",
)

_lib = None


class SimplicialAttnError(RuntimeError):
    pass


def load_library(build: bool = True):
    """Load (building first if stale) the in-tree libsimplicial.so.  Raises if it cannot."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.build() if build else _build.LIB
    if not os.path.exists(path):
        raise SimplicialAttnError(f"libsimplicial.so missing at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P, I, U, S, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_float
    sig = {
        "simplicial_attn_fwd": ([P] * 8 + [S] + [I] * 6 + [U, P], ctypes.c_int),
        "simplicial_attn_fwd_prefixed": ([P] * 8 + [S] + [I] * 7 + [U, P], ctypes.c_int),
        "simplicial_attn_fwd_workspace_bytes": ([I] * 6 + [U], S),
        "simplicial_attn_fwd_workspace_bytes_prefixed": ([I] * 7 + [U], S),
        "simplicial_attn_bwd_workspace_bytes": ([I] * 6 + [U], S),
        "simplicial_attn_bwd_workspace_bytes_prefixed": ([I] * 7 + [U], S),
        "simplicial_attn_bwd": ([P] * 14 + [S] + [I] * 6 + [U, P], ctypes.c_int),
        "simplicial_attn_bwd_prefixed": ([P] * 14 + [S] + [I] * 7 + [U, P], ctypes.c_int),
        "simplicial_attn_host_step_scratch_bytes": ([I] * 6 + [U], S),
        "simplicial_attn_host_step": ([P] * 14 + [S] + [I] * 6 + [U, P], ctypes.c_int),
        "simplicial_attn_fwd_path": ([I] * 6 + [U], ctypes.c_int),
        "simplicial_attn_bwd_path": ([I] * 6 + [U], ctypes.c_int),
        "simplicial_attn_launch_count": ([], ctypes.c_uint64),
        "simplicial_attn_status_string": ([ctypes.c_int], ctypes.c_char_p),
        "simplicial_attn_version": ([], ctypes.c_char_p),
        "simplicial_attn_profile_enable": ([ctypes.c_int], None),
        "simplicial_attn_profile_read": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_int64), ctypes.c_int], ctypes.c_int),
        "simplicial_attn_fwd_gqa_workspace_bytes": ([I] * 7 + [U], S),
        "simplicial_attn_fwd_gqa": ([P] * 8 + [S] + [I] * 7 + [U, P], ctypes.c_int),
        "simplicial_attn_bwd_gqa_workspace_bytes": ([I] * 7 + [U], S),
        "simplicial_attn_bwd_gqa": ([P] * 14 + [S] + [I] * 7 + [U, P], ctypes.c_int),
        "simplicial_attn_fwd_bias_workspace_bytes": ([I] * 7 + [U], S),
        "simplicial_attn_fwd_bias": ([P] * 7 + [F, F, P, S] + [I] * 7 + [U, P], ctypes.c_int),
        "simplicial_attn_bwd_bias_workspace_bytes": ([I] * 7 + [U], S),
        "simplicial_attn_bwd_bias": ([P] * 13 + [F, F, P, S] + [I] * 7 + [U, P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def lib():
    return load_library()


def _check(status: int, what: str):
    if status != 0:
        raise SimplicialAttnError(f"{what} failed: {_STATUS.get(status, status)}")


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _flags(dtype: torch.dtype, det: bool, out_f32: bool, force_simt: bool) -> int:
    f = SA_VARIANT_DET if det else 0
    if dtype == torch.float32:
        f |= SA_IN_F32
    elif dtype != torch.bfloat16:
        raise SimplicialAttnError(f"inputs must be bf16 or fp32, got {dtype}")
    if out_f32:
        f |= SA_OUT_F32
    if force_simt:
        f |= SA_FORCE_SIMT
    return f


def _out_dtype(flags: int) -> torch.dtype:
    return torch.float32 if flags & (SA_IN_F32 | SA_OUT_F32) else torch.bfloat16


def _check_inputs(q, keys, n_prefix, h_kv=None):
    if not q.is_cuda:
        raise SimplicialAttnError("simplicial_attn needs CUDA tensors (there is no CPU path)")
    B, N, H, D = q.shape
    Hk = H if h_kv is None else h_kv
    for t in (q, *keys):
        if not t.is_contiguous() or t.dtype != q.dtype or t.device != q.device:
            raise SimplicialAttnError("inputs must be contiguous, same dtype and device")
    for t in keys:
        if tuple(t.shape) != (B, N + n_prefix, Hk, D):
            raise SimplicialAttnError(f"key-side tensor shape {tuple(t.shape)} != {(B, N + n_prefix, Hk, D)}")
    return B, N, H, D


_ws_cache: dict = {}


def _workspace(device, nbytes: int, kind: str = "fwd") -> torch.Tensor:
    """Per-(device, stream) scratch reused across calls; calls on one stream are ordered, so reuse
    is safe."""
    key = (kind, device.type, device.index, torch.cuda.current_stream(device).cuda_stream)
    t = _ws_cache.get(key)
    if t is None or t.numel() < max(nbytes, 1):
        t = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def forward(q, k, v, k2, v2, w1: int, w2: int, det: bool = False, out_f32: bool = False,
            n_prefix: int = 0, force_simt: bool = False, k2_bias: float = 0.0, v2_bias: float = 0.0):
    """o, lse = 2-simplicial attention forward (simplicial_attn_fwd_prefixed; key-side tensors with
    fewer heads than q -> grouped-query simplicial_attn_fwd_gqa; a nonzero k2_bias / v2_bias ->
    simplicial_attn_fwd_bias)."""
    h_kv = k.shape[2] if k.dim() == 4 and k.shape[2] != q.shape[2] else None
    B, N, H, D = _check_inputs(q, (k, v, k2, v2), n_prefix, h_kv)
    L = lib()
    flags = _flags(q.dtype, det, out_f32, force_simt)
    o = torch.empty((B, N, H, D), dtype=_out_dtype(flags), device=q.device)
    lse = torch.empty((B, H, N), dtype=torch.float32, device=q.device)
    if k2_bias != 0.0 or v2_bias != 0.0:
        if n_prefix:
            raise SimplicialAttnError("the bias entry points take no key prefix")
        hk = h_kv or H
        wsb = int(L.simplicial_attn_fwd_bias_workspace_bytes(B, H, hk, N, D, w1, w2, flags))
        ws = _workspace(q.device, wsb, "fwd_bias")
        st = L.simplicial_attn_fwd_bias(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(o), _ptr(lse),
                                        float(k2_bias), float(v2_bias), _ptr(ws), ws.numel(), B, H, hk, N, D,
                                        w1, w2, flags, _stream(q.device))
        _check(st, "simplicial_attn_fwd_bias")
        return o, lse
    if h_kv is not None:
        if n_prefix:
            raise SimplicialAttnError("grouped-query mode takes no key prefix")
        wsb = int(L.simplicial_attn_fwd_gqa_workspace_bytes(B, H, h_kv, N, D, w1, w2, flags))
        ws = _workspace(q.device, wsb)
        st = L.simplicial_attn_fwd_gqa(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(o), _ptr(lse),
                                       _ptr(ws), ws.numel(), B, H, h_kv, N, D, w1, w2, flags, _stream(q.device))
        _check(st, "simplicial_attn_fwd_gqa")
        return o, lse
    wsb = int(L.simplicial_attn_fwd_workspace_bytes_prefixed(B, H, N, D, w1, w2, n_prefix, flags))
    ws = _workspace(q.device, wsb)
    st = L.simplicial_attn_fwd_prefixed(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(o), _ptr(lse),
                                        _ptr(ws), ws.numel(), B, H, N, D, w1, w2, n_prefix, flags,
                                        _stream(q.device))
    _check(st, "simplicial_attn_fwd")
    return o, lse


def backward(q, k, v, k2, v2, o, lse, dO, w1: int, w2: int, det: bool = False, out_f32: bool = False,
             n_prefix: int = 0, force_simt: bool = False, workspace: torch.Tensor | None = None,
             k2_bias: float = 0.0, v2_bias: float = 0.0):
    """dq, dk, dv, dk2, dv2 = 2-simplicial attention backward (simplicial_attn_bwd_prefixed; key-side
    tensors with fewer heads than q -> grouped-query simplicial_attn_bwd_gqa; a nonzero k2_bias /
    v2_bias -> simplicial_attn_bwd_bias)."""
    h_kv = k.shape[2] if k.dim() == 4 and k.shape[2] != q.shape[2] else None
    B, N, H, D = _check_inputs(q, (k, v, k2, v2), n_prefix, h_kv)
    L = lib()
    flags = _flags(q.dtype, det, out_f32, force_simt)
    od = _out_dtype(flags)
    if o.dtype != od or dO.dtype != q.dtype or not dO.is_contiguous() or not o.is_contiguous():
        raise SimplicialAttnError("o must be in the output dtype and dO in the input dtype, contiguous")
    dq = torch.empty((B, N, H, D), dtype=od, device=q.device)
    dk, dv, dk2, dv2 = (torch.empty_like(k, dtype=od) for _ in range(4))
    if k2_bias != 0.0 or v2_bias != 0.0:
        if n_prefix:
            raise SimplicialAttnError("the bias entry points take no key prefix")
        hk = h_kv or H
        wsb = int(L.simplicial_attn_bwd_bias_workspace_bytes(B, H, hk, N, D, w1, w2, flags))
        ws = _workspace(q.device, wsb, "bwd_bias")
        st = L.simplicial_attn_bwd_bias(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(o), _ptr(lse),
                                        _ptr(dO), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dk2), _ptr(dv2),
                                        float(k2_bias), float(v2_bias), _ptr(ws), ws.numel(), B, H, hk, N, D,
                                        w1, w2, flags, _stream(q.device))
        _check(st, "simplicial_attn_bwd_bias")
        return dq, dk, dv, dk2, dv2
    if h_kv is not None:
        if n_prefix:
            raise SimplicialAttnError("grouped-query mode takes no key prefix")
        wsb = int(L.simplicial_attn_bwd_gqa_workspace_bytes(B, H, h_kv, N, D, w1, w2, flags))
        ws = _workspace(q.device, wsb, "bwd_gqa")
        st = L.simplicial_attn_bwd_gqa(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(o), _ptr(lse),
                                       _ptr(dO), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dk2), _ptr(dv2),
                                       _ptr(ws), ws.numel(), B, H, h_kv, N, D, w1, w2, flags, _stream(q.device))
        _check(st, "simplicial_attn_bwd_gqa")
        return dq, dk, dv, dk2, dv2
    wsb = int(L.simplicial_attn_bwd_workspace_bytes_prefixed(B, H, N, D, w1, w2, n_prefix, flags))
    if workspace is None or workspace.numel() < wsb:
        workspace = _workspace(q.device, wsb, "bwd")
    st = L.simplicial_attn_bwd_prefixed(_ptr(q), _ptr(k), _ptr(v), _ptr(k2), _ptr(v2), _ptr(o), _ptr(lse),
                                        _ptr(dO), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dk2), _ptr(dv2),
                                        _ptr(workspace), workspace.numel(), B, H, N, D, w1, w2, n_prefix,
                                        flags, _stream(q.device))
    _check(st, "simplicial_attn_bwd")
    return dq, dk, dv, dk2, dv2


def host_step(h_in: dict, h_out: dict, w1: int, w2: int, det: bool = False, out_f32: bool = False,
              scratch: torch.Tensor | None = None, device=None):
    """One forward+backward from HOST (pinned) tensors through simplicial_attn_host_step.
    h_in: q,k,v,k2,v2,dO (CPU); h_out: o,lse,dq,dk,dv,dk2,dv2 (CPU, preallocated).
    Returns the device scratch tensor (reuse it across calls)."""
    L = lib()
    q = h_in["q"]
    B, N, H, D = q.shape
    flags = _flags(q.dtype, det, out_f32, False)
    need = int(L.simplicial_attn_host_step_scratch_bytes(B, H, N, D, w1, w2, flags))
    device = device or torch.device("cuda", torch.cuda.current_device())
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(need, dtype=torch.uint8, device=device)
    st = L.simplicial_attn_host_step(*(_ptr(h_in[n]) for n in ("q", "k", "v", "k2", "v2", "dO")),
                                     *(_ptr(h_out[n]) for n in ("o", "lse", "dq", "dk", "dv", "dk2", "dv2")),
                                     _ptr(scratch), scratch.numel(), B, H, N, D, w1, w2, flags,
                                     _stream(device))
    _check(st, "simplicial_attn_host_step")
    return scratch


def fwd_path(B, H, N, D, w1, w2, dtype=torch.bfloat16, det=False, out_f32=False, force_simt=False) -> int:
    return int(lib().simplicial_attn_fwd_path(B, H, N, D, w1, w2, _flags(dtype, det, out_f32, force_simt)))


def bwd_path(B, H, N, D, w1, w2, dtype=torch.bfloat16, det=False, out_f32=False, force_simt=False) -> int:
    return int(lib().simplicial_attn_bwd_path(B, H, N, D, w1, w2, _flags(dtype, det, out_f32, force_simt)))


def launch_count() -> int:
    return int(lib().simplicial_attn_launch_count())


def profile_enable(on: bool = True) -> None:
    """Bracket every library kernel launch with CUDA events on its stream (bench roofline)."""
    lib().simplicial_attn_profile_enable(1 if on else 0)


def profile_read(max_kernels: int = 64) -> dict:
    """{kernel name: (total ms, launches)} recorded since the last read; clears the record."""
    names = ctypes.create_string_buffer(32 * max_kernels)
    tot = (ctypes.c_double * max_kernels)()
    cnt = (ctypes.c_int64 * max_kernels)()
    n = lib().simplicial_attn_profile_read(names, tot, cnt, max_kernels)
    out = {}
    for k in range(n):
        nm = names.raw[32 * k:32 * k + 32].split(b"\0", 1)[0].decode()
        out[nm] = (float(tot[k]), int(cnt[k]))
    return out
