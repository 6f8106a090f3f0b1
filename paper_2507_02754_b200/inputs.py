"""Seeded synthetic inputs and the BASELINE.json configurations.

This module holds NO arithmetic of the method: it only draws random numbers and
names shapes.  It is the one piece shared by the CUDA path's tests/bench and the
oracle's tests.

Recipe: q, k, v, k2, v2, dO are drawn in that fixed order as
float32 N(0,1) ``randn`` from ``torch.Generator(device).manual_seed(seed)``, then
rounded to nearest-even to bf16 (bf16 configs) or kept fp32 (c1).  The oracle
receives exactly these rounded values, upcast to float64.  Key-side tensors
(k, v, k2, v2) carry ``n_prefix`` extra leading rows (sequence-sharded mode).
"""
from __future__ import annotations

import torch

# BASELINE.json "configs", in order (c1..c5).  bwd=False -> forward-only config.
CONFIGS = {
    "c1": dict(B=1, H=1, N=128, D=16, w1=32, w2=8, dtype="f32", det=False, bwd=True),
    "c2": dict(B=1, H=16, N=8192, D=128, w1=512, w2=32, dtype="bf16", det=False, bwd=False),
    "c3": dict(B=4, H=16, N=8192, D=128, w1=512, w2=32, dtype="bf16", det=False, bwd=True),
    "c4": dict(B=2, H=16, N=16384, D=128, w1=512, w2=32, dtype="bf16", det=True, bwd=True),
    "c5": dict(B=8, H=32, N=32768, D=128, w1=1024, w2=64, dtype="bf16", det=False, bwd=True),
}

NAMES = ("q", "k", "v", "k2", "v2", "dO")
KEY_SIDE = ("k", "v", "k2", "v2")


def seed_of(cfg: str, salt: int = 0) -> int:
    """seed = 1000*cfg_index + salt."""
    return 1000 * int(cfg.lstrip("c")) + salt


def torch_dtype(name: str) -> torch.dtype:
    return {"f32": torch.float32, "bf16": torch.bfloat16}[name]


def make_inputs(B: int, N: int, H: int, D: int, seed: int, dtype: str = "bf16",
                n_prefix: int = 0, device: str = "cpu", names=NAMES) -> dict:
    """Draw the inputs.  Returns {name: tensor[B, rows, H, D]} in ``dtype`` on ``device``;
    rows = N for q/dO and n_prefix+N for key-side tensors."""
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    out = {}
    for name in NAMES:
        rows = N + n_prefix if name in KEY_SIDE else N
        t = torch.randn((B, rows, H, D), generator=gen, dtype=torch.float32, device=device)
        if name in names:
            out[name] = t.to(torch_dtype(dtype)).contiguous()
    return out
