"""GQA timing: B=1, H query heads sharing H_kv key heads, c3 windows; fwd+bwd ms vs the MHA run
with the same query heads (the expand-and-reduce GQA backward adds fp32 partials + one reduction)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_02754_b200 as sa

def run(B, H, Hk, N, D, w1, w2, steps=5):
    g = torch.Generator().manual_seed(0)
    q, dO = (torch.randn(B, N, H, D, generator=g).to(torch.bfloat16).cuda() for _ in range(2))
    keys = [torch.randn(B, N, Hk, D, generator=g).to(torch.bfloat16).cuda() for _ in range(4)]
    for _ in range(2):
        o, lse = sa.forward(q, *keys, w1, w2)
        sa.backward(q, *keys, o, lse, dO, w1, w2)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(steps):
        o, lse = sa.forward(q, *keys, w1, w2)
    e[1].record()
    for _ in range(steps):
        sa.backward(q, *keys, o, lse, dO, w1, w2)
    e[2].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / steps, e[1].elapsed_time(e[2]) / steps

N, D, w1, w2 = 8192, 128, 512, 32
for H, Hk in ((64, 64), (64, 8), (64, 1)):
    f, b = run(1, H, Hk, N, D, w1, w2)
    fl = 27 * 1 * H * N * w1 * w2 * D
    print(json.dumps({"B": 1, "H": H, "H_kv": Hk, "N": N, "w1": w1, "w2": w2, "fwd_ms": f, "bwd_ms": b,
                      "tflops_paper_basis": fl / ((f + b) / 1e3) / 1e12}))
