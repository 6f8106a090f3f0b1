"""(GPU box) Forward window-split check: CUDA forward vs the oracle for a list of window shapes,
printing the per-query error pattern (which queries / positions are off)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2507_02754_b200 as sa  # noqa: E402
from paper_2507_02754_b200.inputs import make_inputs  # noqa: E402

shapes = [(1, 200, 1, 128, 40, 64), (1, 200, 1, 128, 64, 40), (1, 200, 1, 128, 64, 48), (1, 200, 1, 128, 64, 64),
          (1, 200, 1, 128, 128, 128), (1, 200, 1, 128, 64, 100)]
for (B, N, H, D, w1, w2) in shapes:
    inp = make_inputs(B, N, H, D, seed=7 * N + D, dtype="bf16")
    t = {n: x.cuda() for n, x in inp.items()}
    o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, out_f32=True)
    torch.cuda.synchronize()
    a = {n: x.double().numpy() for n, x in inp.items()}
    ro, rl = oracle.forward(a["q"], a["k"], a["v"], a["k2"], a["v2"], w1, w2)
    eo = np.abs(o.double().cpu().numpy() - ro).max(axis=(0, 2, 3))
    el = np.abs(lse.double().cpu().numpy() - rl).max(axis=(0, 1))
    bad = np.nonzero(~(eo < 2e-2) | ~(el < 2e-2))[0]
    print((w1, w2), "o err", float(np.nanmax(eo)), "lse err", float(np.nanmax(el)), "bad queries", bad[:20], len(bad))
    if len(bad):
        i = bad[0]
        print("  lse got", lse[0, 0, i - 2:i + 3].tolist(), "ref", rl[0, 0, i - 2:i + 3].tolist())
