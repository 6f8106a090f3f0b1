"""torch.autograd wrapper around the C-ABI forward/backward (the training
interface; the paper interleaves 2-simplicial layers every 4th block).

``simplicial_attention(q, k, v, k2, v2, w1, w2)`` returns o [B,N,H,D]; its backward calls
``simplicial_attn_bwd`` with the forward's stored o and lse (reading R23).  Argument marshalling
only: every step of forward and backward runs in libsimplicial.so; there is no CPU path.
Inputs are bf16 (tcgen05 path) or fp32 (exact CUDA-core path), layout [B,N,H,D] (keys
[B,N,H,D] too: n_prefix = 0).  Gradients come back in the input dtype.
"""
from __future__ import annotations

import torch

from . import binding


class SimplicialAttnFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, k2, v2, w1: int, w2: int, det: bool):
        q, k, v, k2, v2 = (t.contiguous() for t in (q, k, v, k2, v2))
        o, lse = binding.forward(q, k, v, k2, v2, w1, w2, det=det)
        ctx.save_for_backward(q, k, v, k2, v2, o, lse)
        ctx.w = (w1, w2, det)
        return o

    @staticmethod
    def backward(ctx, dO):
        q, k, v, k2, v2, o, lse = ctx.saved_tensors
        w1, w2, det = ctx.w
        dq, dk, dv, dk2, dv2 = binding.backward(q, k, v, k2, v2, o, lse, dO.contiguous().to(q.dtype), w1, w2,
                                                det=det)
        return dq, dk, dv, dk2, dv2, None, None, None


def simplicial_attention(q, k, v, k2, v2, w1: int, w2: int, det: bool = False):
    """o = sliding-window 2-simplicial attention (Eq. P:230-244; det: P:291-301), differentiable."""
    return SimplicialAttnFunction.apply(q, k, v, k2, v2, w1, w2, det)
