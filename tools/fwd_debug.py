"""Diagnostics: tcgen05 forward vs oracle on small shapes, per-row error summary."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2507_02754_b200 as sa
from paper_2507_02754_b200.inputs import make_inputs

def run(B, N, H, D, w1, w2, det=False):
    inp = make_inputs(B, N, H, D, seed=1, dtype="bf16")
    t = {n: x.cuda() for n, x in inp.items()}
    o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=det, out_f32=True)
    torch.cuda.synchronize()
    a = {n: x.double().numpy() for n, x in inp.items()}
    ro, rl = oracle.forward(a["q"], a["k"], a["v"], a["k2"], a["v2"], w1, w2, det=det)
    eo = np.abs(o.double().cpu().numpy() - ro).max(axis=(0, 2, 3))
    el = np.abs(lse.double().cpu().numpy() - rl).max(axis=(0, 1))
    print(f"B={B} N={N} H={H} D={D} w=({w1},{w2}) det={det}: o err max {eo.max():.3e} lse err max {el.max():.3e}")
    bad = np.where((eo > 2e-2) | (el > 2e-2))[0]
    if len(bad):
        print("  bad rows:", bad[:20], "... n=", len(bad))
        print("  lse got", lse[0, 0, bad[:4]].tolist(), "ref", rl[0, 0, bad[:4]].tolist())
        print("  o got", o[0, bad[0], 0, :6].tolist(), "ref", ro[0, bad[0], 0, :6].tolist())

if __name__ == "__main__":
    for args in [(1, 4, 1, 128, 1, 1), (1, 8, 1, 128, 4, 4), (1, 128, 1, 128, 32, 32), (1, 256, 1, 128, 128, 32),
                 (1, 384, 2, 128, 200, 32), (1, 300, 1, 64, 48, 16), (1, 200, 1, 128, 40, 64)]:
        try:
            run(*args)
        except Exception as e:
            print("ERROR", args, e)
            break
    run(1, 256, 1, 128, 64, 32, det=True)
