"""Run one c3 fwd+bwd with the trace library and print CTA-0 phase timelines (cycles)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_02754_b200 import binding
from paper_2507_02754_b200.inputs import CONFIGS, make_inputs
binding._lib = None
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2507_02754_b200", "libsimplicial_trace.so"))
binding._lib = None
orig = binding._build.build
binding._build.build = lambda *a, **k: os.path.join(ROOT, "paper_2507_02754_b200", "libsimplicial_trace.so")
L = binding.load_library()
L.simplicial_attn_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = dict(CONFIGS[cfg])
for kv in sys.argv[2:]:  # overrides, e.g. w2=64
    k_, v_ = kv.split("=")
    c[k_] = int(v_)
inp = make_inputs(c["B"], c["N"], c["H"], c["D"], 1, dtype=c["dtype"])
t = {n: x.cuda() for n, x in inp.items()}
for rep in range(2):
    buf = (ctypes.c_ulonglong * 8192)()
    L.simplicial_attn_debug_trace(buf, 4096)
    o, lse = binding.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], c["w1"], c["w2"], det=c["det"])
    torch.cuda.synchronize()
    n = L.simplicial_attn_debug_trace(buf, 4096)
    fwd = [(buf[2 * i], buf[2 * i + 1], i // 512) for i in range(4096) if buf[2 * i + 1]]
    binding.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], c["w1"], c["w2"], det=c["det"])
    torch.cuda.synchronize()
    n = L.simplicial_attn_debug_trace(buf, 4096)
    bwd = [(buf[2 * i], buf[2 * i + 1], i // 512) for i in range(4096) if buf[2 * i + 1]]
for name, ev in (("fwd", fwd), ("bwd", bwd)):
    if not ev:
        continue
    ev.sort(key=lambda x: x[1])
    t0 = ev[0][1]
    print(f"== {name}: {len(ev)} events")
    for tag, clk, reg in ev[:400]:
        print(f"  {clk - t0:9d}  r{reg} item {tag >> 16}  tag {(tag >> 8) & 0xff:3d}  c {tag & 0xff}")
