"""Diagnostics: tensor-core backward vs oracle on small shapes, per-tensor error summary."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2507_02754_b200 as sa
from paper_2507_02754_b200.inputs import make_inputs

def run(B, N, H, D, w1, w2, det=False):
    inp = make_inputs(B, N, H, D, seed=2, dtype="bf16")
    t = {n: x.cuda() for n, x in inp.items()}
    o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=det, out_f32=True)
    g = sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2, det=det, out_f32=True)
    torch.cuda.synchronize()
    a = {n: x.double().numpy() for n, x in inp.items()}
    rg = oracle.backward(a["q"], a["k"], a["v"], a["k2"], a["v2"], a["dO"], w1, w2, det=det)
    path = sa.bwd_path(B, H, N, D, w1, w2, det=det, out_f32=True)
    msg = []
    for n, x, r in zip(("dq", "dk", "dv", "dk2", "dv2"), g, rg):
        e = np.abs(x.double().cpu().numpy() - r)
        rows = e.max(axis=(0, 2, 3))
        bad = np.where(rows > 2e-2)[0]
        msg.append(f"{n}={e.max():.2e}" + (f"[bad rows {bad[:8].tolist()} n={len(bad)}]" if len(bad) else ""))
    print(f"path={path} B={B} N={N} H={H} D={D} w=({w1},{w2}) det={det}: " + " ".join(msg), flush=True)

if __name__ == "__main__":
    for args in [(1, 8, 1, 128, 4, 4), (1, 128, 1, 128, 32, 32), (1, 256, 1, 128, 128, 32), (1, 384, 2, 128, 200, 32),
                 (1, 300, 1, 64, 48, 16), (1, 200, 1, 128, 40, 64), (2, 1000, 2, 128, 64, 32)]:
        run(*args)
    run(1, 256, 1, 128, 64, 32, det=True)
    run(1, 160, 1, 128, 16, 48, det=True)
