"""Run one c3 backward with the trace library and print the bwd_q pair kernel's phase timeline
(cluster 0, three steady-state tiles; regions 4*rank + role: 0 MMA, 1 softmax warp, 2 epilogue, 3 TMA)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_02754_b200 import binding
from paper_2507_02754_b200.inputs import CONFIGS, make_inputs
binding._build.build = lambda *a, **k: os.path.join(ROOT, "paper_2507_02754_b200", "libsimplicial_trace.so")
binding._lib = None
L = binding.load_library()
L.simplicial_attn_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
c = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
inp = make_inputs(c["B"], c["N"], c["H"], c["D"], 1, dtype=c["dtype"])
t = {n: x.cuda() for n, x in inp.items()}
o, lse = binding.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], c["w1"], c["w2"], det=c["det"])
buf = (ctypes.c_ulonglong * 8192)()
for rep in range(2):
    L.simplicial_attn_debug_trace(buf, 4096)
    binding.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], c["w1"], c["w2"], det=c["det"])
    torch.cuda.synchronize()
    L.simplicial_attn_debug_trace(buf, 4096)
idx = [b * 256 + i for b in (0, 1, 2, 3, 4, 5, 14, 15) for i in range(255)]
ev = [(buf[2 * i], buf[2 * i + 1]) for i in idx if buf[2 * i + 1]]
ev.sort(key=lambda x: x[1])
t0 = ev[0][1]
role = ["MMA", "SMX", "EPI", "TMA"]
print(f"{len(ev)} events")
for tag, clk in ev:
    rg = tag >> 24
    print(f"{clk - t0:9d}  r{rg // 4} {role[rg % 4]}  tile {(tag >> 16) & 0xff}  ev {(tag >> 8) & 0xff:3d}  c {tag & 0xff}")
