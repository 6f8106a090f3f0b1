"""torch.autograd wrapper around the C-ABI forward/backward (the training
interface; the paper interleaves 2-simplicial layers every 4th block).

``simplicial_attention(q, k, v, k2, v2, w1, w2)`` returns o [B,N,H,D]; its backward calls
``simplicial_attn_bwd`` with the forward's stored o and lse (reading R23).  Argument marshalling
only: every step of forward and backward runs in libsimplicial.so; there is no CPU path.
Inputs are bf16 (tcgen05 path) or fp32 (exact CUDA-core path), layout [B,N,H,D] (keys
[B,N,H,D], or [B,N,H_kv,D] for grouped-query heads: n_prefix = 0).  Gradients come back in the
input dtype.  Optional scalar k2_bias / v2_bias go to the bias entry points.
"""
from __future__ import annotations

import torch

from . import binding


class SimplicialAttnFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, k2, v2, w1: int, w2: int, det: bool, k2_bias: float = 0.0, v2_bias: float = 0.0):
        q, k, v, k2, v2 = (t.contiguous() for t in (q, k, v, k2, v2))
        o, lse = binding.forward(q, k, v, k2, v2, w1, w2, det=det, k2_bias=k2_bias, v2_bias=v2_bias)
        ctx.save_for_backward(q, k, v, k2, v2, o, lse)
        ctx.w = (w1, w2, det, k2_bias, v2_bias)
        return o

    @staticmethod
    def backward(ctx, dO):
        q, k, v, k2, v2, o, lse = ctx.saved_tensors
        w1, w2, det, k2_bias, v2_bias = ctx.w
        dq, dk, dv, dk2, dv2 = binding.backward(q, k, v, k2, v2, o, lse, dO.contiguous().to(q.dtype), w1, w2,
                                                det=det, k2_bias=k2_bias, v2_bias=v2_bias)
        return dq, dk, dv, dk2, dv2, None, None, None, None, None


def simplicial_attention(q, k, v, k2, v2, w1: int, w2: int, det: bool = False, k2_bias: float = 0.0,
                         v2_bias: float = 0.0):
    """o = sliding-window 2-simplicial attention (Eq. P:230-244; det: P:291-301), differentiable.
    k2_bias / v2_bias: the scalars the paper's kernel adds to the K' / V' tiles."""
    return SimplicialAttnFunction.apply(q, k, v, k2, v2, w1, w2, det, k2_bias, v2_bias)
