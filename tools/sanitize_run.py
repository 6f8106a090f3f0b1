#!/usr/bin/env python
"""Small forward+backward runs of every tensor-core kernel variant, for compute-sanitizer
(memcheck / racecheck / synccheck; tests/test_sanitizer.py).  Covers tc_fwd, tc_delta, tc_cvt_f16,
tc_bwd_q (R = 32 row-owned epilogue, R = 64, R = 128 shared/global ring, R = 8 generic, det passes),
tc_fold and tc_bwd_kv, plus the fp32 CUDA-core kernels.  Exits non-zero on a CUDA error; results are
not checked here (the parity tests do that)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_02754_b200 import binding as sa  # noqa: E402
from paper_2507_02754_b200.inputs import make_inputs  # noqa: E402

CASES = [
    # B, N, H, D, w1, w2, det, dtype
    (1, 300, 1, 128, 128, 32, False, "bf16"),   # R = 32 rotated epilogue (c3 tiling), 2 CTA ranges
    (1, 300, 1, 128, 128, 32, True, "bf16"),    # det R = 32
    (1, 200, 1, 128, 96, 64, False, "bf16"),    # R = 64
    (1, 160, 1, 128, 128, 128, False, "bf16"),  # R = 128 trilinear (shared ring, G = 1)
    (1, 160, 1, 128, 128, 128, True, "bf16"),   # R = 128 det (global ring)
    (1, 200, 1, 64, 32, 8, False, "bf16"),      # R = 8 generic passes, D = 64
    (1, 130, 1, 128, 40, 24, False, "bf16"),    # R = 24 forward / padded 32 backward
    (1, 96, 1, 16, 32, 8, False, "f32"),        # fp32 CUDA-core path
]


def main():
    which = sys.argv[1:] or [str(i) for i in range(len(CASES))]
    dev = torch.device("cuda", 0)
    for idx in map(int, which):
        B, N, H, D, w1, w2, det, dt = CASES[idx]
        inp = make_inputs(B, N, H, D, seed=idx, dtype=dt)
        t = {n: x.to(dev) for n, x in inp.items()}
        o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=det, out_f32=True)
        g = sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2, det=det, out_f32=True)
        torch.cuda.synchronize()
        assert all(torch.isfinite(x).all() for x in (o, lse, *g)), CASES[idx]
        print("case", idx, CASES[idx], "ok", flush=True)


if __name__ == "__main__":
    main()
