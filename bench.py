#!/usr/bin/env python
"""Benchmark: sliding-window 2-simplicial attention fwd+bwd on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

A "step" is one forward + backward (every hot-path kernel) over one batch of synthetic
inputs of BASELINE config c3 (B=4 H=16 N=8192 D=128 w1=512 w2=32, bf16 in) -- the
configuration the metric's >=50%-of-peak target is quoted on.  N>1 runs under torchrun, one
process per GPU: each rank processes its own c3-sized B*H shard (weak scaling, no data-path
collective; NCCL only for the barrier and the max-over-ranks timing).

FLOP bases:
  paper formula (value): fwd 6*NW*D (Sec. 6), bwd 21*NW*D (7 backward einsums P:393-413
      at the same 3-flop convention), NW = B*H*N*w1*w2 nominal triples;
  tensor-core MMA (roofline): fwd 4*NW*D, bwd 14*NW*D (each einsum is one 2-flop contraction).
``--impl reference`` times the float64 CPU oracle (oracle/) on a bounded sample of the same
workload -- the reference arm of this tier (there is no runnable reference implementation).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_02754_b200.inputs import CONFIGS, make_inputs, seed_of  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

PAPER_FLOPS_PER_TRIPLE_D = {"fwd": 6, "bwd": 21}
MMA_FLOPS_PER_TRIPLE_D = {"fwd": 4, "bwd": 14}


def peaks():
    if os.path.exists(PEAKS_PATH):
        p = json.load(open(PEAKS_PATH))
        return p, "measured"
    return FALLBACK_PEAKS, "fallback"


def nominal_triples(c):
    return c["B"] * c["H"] * c["N"] * c["w1"] * c["w2"]


def paper_flops(c, which=("fwd", "bwd")):
    return sum(PAPER_FLOPS_PER_TRIPLE_D[w] for w in which) * nominal_triples(c) * c["D"]


# Algorithmic work of each library kernel per launch on config c:
# (bound, unit, amount).  Tensor-core kernels: MMA flops of the contractions they own;
# SIMT kernels: fp32 flops of the same contractions on CUDA cores ("alu");
# delta pre-pass: bytes (hbm).
def kernel_work(name: str, c: dict, out_bytes: int):
    T, D = nominal_triples(c), c["D"]
    rows = c["B"] * c["H"] * c["N"]
    table = {
        "tc_fwd": ("tensor", 4 * T * D),            # S = A K^T and U = P V
        "tc_bwd_kv": ("tensor", 8 * T * D),         # S, dP recompute; dV += P A_dP; dK += dS A_S
        "tc_bwd_q": ("tensor", 8 * T * D),          # S, dP recompute; W = dS K; U = P V
        "simt_fwd": ("alu", 4 * T * D),
        "simt_bwd_dq": ("alu", 6 * T * D),
        "simt_bwd_dk2": ("alu", 8 * T * D),
        "simt_bwd_dk": ("alu", 8 * T * D),
        "simt_delta": ("hbm", rows * D * (2 + out_bytes) + rows * 4),
        "tc_delta": ("hbm", rows * D * (2 + out_bytes) + rows * 4),
    }
    return table.get(name)


def kernel_traffic(name: str, c: dict):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of `name` from the
    newest committed `ncu --set full` summary for this config (profiles/*_traffic_<cfg>.json,
    written by tools/profile_summarize.py), or (None, reason)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_traffic_{c['name']}.json")))  # newest tag sorts last
    for fn in reversed(files):
        k = json.load(open(fn)).get("kernels", {}).get(name)
        if k:
            return k["traffic_bytes"], f"profiles/{os.path.basename(fn)} (one ncu --set full capture)"
    return None, "no ncu --set full capture committed for this config"


def alu_peak_tflops(sm_mhz: float) -> float:
    """fp32 FMA peak: 148 SMs x 128 FP32 lanes x 2 flop x clock."""
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [ln.split(",") for ln in open(self.f.name).read().strip().splitlines() if ln.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------------------------
# Reference arm / cpu_baseline: the float64 oracle on a bounded, window-exact sample.
# --------------------------------------------------------------------------------------------
def oracle_sample(c, seed, L):
    """Queries [a, a+L) of slice (b=0, h=0) with the (max(w1,w2)-1)-row key halo as prefix, so
    every sampled row sees its full window: oracle fwd+bwd.  Returns (seconds, paper flops)."""
    import numpy as np

    import oracle
    N, D, w1, w2 = c["N"], c["D"], c["w1"], c["w2"]
    npf = max(w1, w2) - 1
    a = min(N - L, max(npf, N // 2))
    g = torch.Generator().manual_seed(seed)
    shape_q, shape_k = (1, L, 1, D), (1, L + npf, 1, D)
    dt = torch.float32 if c["dtype"] == "f32" else torch.bfloat16
    t = {n: torch.randn(shape_k if n in ("k", "v", "k2", "v2") else shape_q, generator=g).to(dt).double().numpy()
         for n in ("q", "k", "v", "k2", "v2", "dO")}
    t0 = time.perf_counter()
    oracle.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=c["det"], n_prefix=npf)
    if c["bwd"]:
        oracle.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], t["dO"], w1, w2, det=c["det"], n_prefix=npf)
    dt_s = time.perf_counter() - t0
    which = ("fwd", "bwd") if c["bwd"] else ("fwd",)
    flops = sum(PAPER_FLOPS_PER_TRIPLE_D[w] for w in which) * L * w1 * w2 * D
    del np, a
    return dt_s, flops


def calibrate_oracle_rows(c, target_s):
    import oracle
    oracle.build()
    # two-point calibration: the halo makes the cost affine in L (t = a + b L)
    L0, L1 = 32, 160
    t0, _ = oracle_sample(c, 0, L0)
    t1, _ = oracle_sample(c, 0, L1)
    b = max((t1 - t0) / (L1 - L0), 1e-6)
    a = max(t0 - b * L0, 0.0)
    L = int(min(c["N"] - 1, max(L0, (target_s - a) / b)))
    return L


def cpu_baseline(c, target_s=15.0):
    import oracle
    L = calibrate_oracle_rows(c, target_s)
    secs, flops = oracle_sample(c, 1, L)
    return {"value": flops / secs / 1e12, "unit": "TFLOP/s", "cores": oracle.threads_used(),
            "kind": "oracle",
            "sample": f"float64 C oracle, fwd+bwd of {L} query rows (b=0,h=0) with a "
                      f"{max(c['w1'], c['w2']) - 1}-row key halo of config {c['name']}, {secs:.1f} s; "
                      f"paper-formula FLOPs of the sample / wall time"}


def run_reference(args, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    L = calibrate_oracle_rows(c, target_s=max(2.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(c, 2, L)
    tot_s, tot_f = 0.0, 0.0
    for s in range(args.steps):
        secs, fl = oracle_sample(c, 3 + s, L)
        tot_s += secs
        tot_f += fl
    val = tot_f / tot_s / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(c, args.gpus),
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": oracle.threads_used(), "kind": "oracle",
                         "sample": f"each step: fwd+bwd of {L} query rows (b=0,h=0, full key halo) of "
                                   f"config {c['name']}"},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# Table 1 of the paper: latency of the (w1, w2) pairs it reports, on its (unstated) shape.
TABLE1 = [(1024, 32, 104.1), (512, 64, 110.7), (128, 128, 59.2), (256, 64, 55.8), (512, 32, 55.1),
          (1024, 16, 55.1), (256, 32, 28.3)]


def run_table1(args, c):
    """Re-measure the paper's only kernel experiment on B200: fwd+bwd latency and TFLOP/s (paper
    basis) of each (w1, w2) pair at config c's B, H, N, D; the paper's ms are quoted as context
    (their shape and hardware are not stated, so they are not a like-for-like baseline)."""
    import paper_2507_02754_b200 as sa
    dev = torch.device("cuda", 0)
    B, H, N, D, det = (c[k] for k in ("B", "H", "N", "D", "det"))
    inp = make_inputs(B, N, H, D, seed_of(args.config), dtype=c["dtype"], device="cpu")
    t = {n: x.to(dev) for n, x in inp.items()}
    stream = torch.cuda.current_stream(dev)
    for w1, w2, paper_ms in TABLE1:
        cc = dict(c, w1=w1, w2=w2)

        def fwd():
            return sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=det)

        def bwd(o, lse):
            sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2, det=det)

        steps = max(1, args.steps)
        for _ in range(max(1, args.warmup)):
            o, lse = fwd()
            bwd(o, lse)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        fms = bms = 0.0
        for _ in range(steps):
            e[0].record(stream)
            o, lse = fwd()
            e[1].record(stream)
            bwd(o, lse)
            e[2].record(stream)
            torch.cuda.synchronize()
            fms += e[0].elapsed_time(e[1])
            bms += e[1].elapsed_time(e[2])
        fms, bms = fms / steps, bms / steps
        # per-kernel split of one more fwd+bwd (library CUDA-event profiling)
        sa.profile_read()
        sa.profile_enable(True)
        o, lse = fwd()
        bwd(o, lse)
        torch.cuda.synchronize()
        kern = {n: round(v[0], 3) for n, v in sa.profile_read().items()}
        sa.profile_enable(False)
        fl = paper_flops(cc)
        print(json.dumps({
            "sweep": "table1", "w1": w1, "w2": w2, "w1xw2": w1 * w2,
            "config": f"B={B} H={H} N={N} D={D} {'det' if det else 'trilinear'} bf16",
            "fwd_ms": fms, "bwd_ms": bms, "ms_per_step": fms + bms,
            "tflops_paper_basis": fl / ((fms + bms) / 1e3) / 1e12,
            "fwd_tflops": paper_flops(cc, ("fwd",)) / (fms / 1e3) / 1e12,
            "paths": {"fwd": {1: "simt", 2: "tcgen05"}.get(sa.fwd_path(B, H, N, D, w1, w2, det=det)),
                      "bwd": {1: "simt", 2: "tcgen05"}.get(sa.bwd_path(B, H, N, D, w1, w2, det=det))},
            "kernels_ms": kern,
            "paper_latency_ms": paper_ms, "paper_note": "paper's shape/hardware unstated (P:335-354); context only",
        }), flush=True)


def run_membound(args, c):
    """The memory-bound small-window point of SURVEY.md §8(d): windows (32, 8) at config c's shape,
    MMA intensity w1*w2/3 = 85 flop/B, below the B200 ridge.  Reports achieved HBM GB/s on the
    algorithmic bytes per (b,h,query row): forward 12*D+4 (q,k,v,k2,v2 read, o written at 2 B/elt,
    lse fp32), backward 24*D+8 (q,k,v,k2,v2,o,dO read, five gradients written, lse and delta),
    against the measured HBM copy bandwidth."""
    import paper_2507_02754_b200 as sa
    dev = torch.device("cuda", 0)
    B, H, N, D = (c[k] for k in ("B", "H", "N", "D"))
    w1, w2 = 32, 8
    inp = make_inputs(B, N, H, D, seed_of(args.config), dtype="bf16", device="cpu")
    t = {n: x.to(dev) for n, x in inp.items()}
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(1, args.warmup)):
        o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2)
        sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    steps = max(1, args.steps)
    torch.cuda.synchronize()
    e[0].record(stream)
    for _ in range(steps):
        o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2)
    e[1].record(stream)
    for _ in range(steps):
        sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2)
    e[2].record(stream)
    torch.cuda.synchronize()
    fms, bms = e[0].elapsed_time(e[1]) / steps, e[1].elapsed_time(e[2]) / steps
    # per-kernel split of one more fwd+bwd (library CUDA-event profiling)
    sa.profile_read()
    sa.profile_enable(True)
    o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2)
    sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2)
    torch.cuda.synchronize()
    kern = {n: round(v[0], 3) for n, v in sa.profile_read().items()}
    sa.profile_enable(False)
    rows = B * H * N
    fb, bb = rows * (12 * D + 4), rows * (24 * D + 8)
    pk, src = peaks()
    cc = dict(c, w1=w1, w2=w2)
    print(json.dumps({
        "sweep": "membound", "config": f"B={B} H={H} N={N} D={D} w1={w1} w2={w2} trilinear bf16",
        "fwd_ms": fms, "bwd_ms": bms, "fwd_gbs": fb / (fms / 1e3) / 1e9, "bwd_gbs": bb / (bms / 1e3) / 1e9,
        "hbm_peak_gbs": pk["hbm_gbs"], "peak_source": src,
        "fwd_frac": fb / (fms / 1e3) / 1e9 / pk["hbm_gbs"], "bwd_frac": bb / (bms / 1e3) / 1e9 / pk["hbm_gbs"],
        "tflops_paper_basis": paper_flops(cc) / ((fms + bms) / 1e3) / 1e12,
        "paths": {"fwd": {1: "simt", 2: "tcgen05"}.get(sa.fwd_path(B, H, N, D, w1, w2)),
                  "bwd": {1: "simt", 2: "tcgen05"}.get(sa.bwd_path(B, H, N, D, w1, w2))},
        "kernels_ms": kern,
    }), flush=True)


def config_block(c, n, mode="bh", scaling="weak"):
    per = "per GPU" if scaling == "weak" else f"sharded over {n} GPU(s)"
    return {"workload": f"{c['name']}: B={c['B']} H={c['H']} N={c['N']} D={c['D']} w1={c['w1']} w2={c['w2']} "
                        f"{'det' if c['det'] else 'trilinear'} {'fwd+bwd' if c['bwd'] else 'fwd'} {per}",
            "B": c["B"], "H": c["H"], "N": c["N"], "D": c["D"], "w1": c["w1"], "w2": c["w2"],
            "variant": "det" if c["det"] else "trilinear",
            "global_batch_heads": c["B"] * c["H"] * (n if scaling == "weak" else 1),
            "seq_len": c["N"], "parallelism": f"{mode}-sharded x{n}",
            "l2": "inputs larger than L2 (no flush): %.0f MB of inputs per step" % (
                6 * c["B"] * c["N"] * c["H"] * c["D"] * 2 / 1e6),
            "flop_basis": "paper formula: fwd 6*NW*D + bwd 21*NW*D, NW = B*H*N*w1*w2"}


# --------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--out-f32", action="store_true", help="write o/grads in fp32 (parity runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", default=None, choices=["table1", "membound"],
                    help="table1: the paper's (w1, w2) latency sweep (Table 1, P:335-354) at the chosen "
                         "config's B, H, N, D; one JSON line per pair (not the bench line)")
    ap.add_argument("--mode", default="bh", choices=["bh", "seq"],
                    help="bh: B*H sharding, no data-path collective; seq: the sequence is split across "
                         "ranks with the NCCL halo exchange (parallel.seq_forward / seq_backward)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="weak: every rank runs a whole config-sized problem of its own (c2-c4 default); "
                         "strong: ONE config-sized problem (global seed) is sharded over the ranks -- "
                         "parallel.bh_slice blocks in bh mode, N/world query rows in seq mode (c5 default, "
                         "the long-context config BASELINE.json shards at 2/4/8 GPUs)")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config], name=args.config)

    if args.impl == "reference":
        run_reference(args, c)
        return
    if args.sweep == "table1":
        run_table1(args, c)
        return
    if args.sweep == "membound":
        run_membound(args, c)
        return

    import paper_2507_02754_b200 as sa
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus or (world == 1 and args.gpus == 1), "launch N>1 under torchrun"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    sa.load_library(build=(rank == 0))
    if world > 1:
        dist.barrier()
    scaling = args.scaling or ("strong" if args.config == "c5" else "weak")
    if args.mode == "seq":
        scaling = "strong" if args.scaling is None else scaling
    B, H, N, D, w1, w2, det = (c[k] for k in ("B", "H", "N", "D", "w1", "w2", "det"))
    shard_desc = None
    if scaling == "weak":
        inp = make_inputs(B, N, H, D, seed_of(args.config, salt=rank), dtype=c["dtype"], device="cpu")
        t = {n: x.to(dev) for n, x in inp.items()}
    else:
        # one global problem (global seed, drawn on the device -- the recipe's Generator(device)), each
        # rank keeps its block: sharded and unsharded runs see identical data
        from paper_2507_02754_b200 import parallel
        full = make_inputs(B, N, H, D, seed_of(args.config), dtype=c["dtype"], device=str(dev))
        if args.mode == "seq":
            lo, hi, _ = parallel.seq_shard(N, rank, world, max(w1, w2) - 1)
            t = {n: x[:, lo:hi].contiguous() for n, x in full.items()}
            shard_desc = f"queries/keys [{lo}, {hi}) of N={N}"
            N = hi - lo
        else:
            b0, b1, h0, h1 = parallel.bh_slice(B, H, rank, world)
            t = {n: x[b0:b1, :, h0:h1].contiguous() for n, x in full.items()}
            shard_desc = f"b [{b0}, {b1}) x h [{h0}, {h1}) of B={B} H={H}"
            B, H = b1 - b0, h1 - h0
        del full
        torch.cuda.empty_cache()
        inp = {n: x.cpu() for n, x in t.items()} if not args.no_e2e else None
    cl = dict(c, B=B, H=H, N=N)  # this rank's problem
    out_bytes = 4 if args.out_f32 else 2
    ws = None
    o = lse = None

    def step():
        nonlocal o, lse, ws
        if args.mode == "seq" and world > 1:
            from paper_2507_02754_b200 import parallel
            o, lse, ext = parallel.seq_forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, sa.forward,
                                               det=det, out_f32=args.out_f32)
            if c["bwd"]:
                parallel.seq_backward(t["q"], ext, o, lse, t["dO"], w1, w2, sa.backward, det=det,
                                      out_f32=args.out_f32)
            return
        o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=det, out_f32=args.out_f32)
        if c["bwd"]:
            sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2, det=det,
                        out_f32=args.out_f32, workspace=ws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region: K full steps ----------------
    clocks = ClockSampler(local)
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = sa.launch_count()
    sa.profile_enable(True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    sa.profile_enable(False)
    launches = sa.launch_count() - launches0
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    prof = sa.profile_read()
    if dist:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    which = ("fwd", "bwd") if c["bwd"] else ("fwd",)
    # whole-job work per step: weak = every rank a whole config problem; strong = one problem
    jobs = world if scaling == "weak" else 1
    flops_step = paper_flops(c, which) * jobs
    value = flops_step * args.steps / (ms / 1e3) / 1e12
    mma_flops_step = sum(MMA_FLOPS_PER_TRIPLE_D[w] for w in which) * nominal_triples(c) * D * jobs

    # ---------------- fwd-only and bwd-only timings (separate loops, this rank's problem) ----------------
    extra = {}
    if c["bwd"] and args.mode == "bh":
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        e[0].record(stream)
        for _ in range(args.steps):
            o, lse = sa.forward(t["q"], t["k"], t["v"], t["k2"], t["v2"], w1, w2, det=det, out_f32=args.out_f32)
        e[1].record(stream)
        e[2].record(stream)
        for _ in range(args.steps):
            sa.backward(t["q"], t["k"], t["v"], t["k2"], t["v2"], o, lse, t["dO"], w1, w2, det=det,
                        out_f32=args.out_f32)
        e[3].record(stream)
        torch.cuda.synchronize()
        fms, bms = e[0].elapsed_time(e[1]) / args.steps, e[2].elapsed_time(e[3]) / args.steps
        extra = {"fwd_tflops": paper_flops(cl, ("fwd",)) / (fms / 1e3) / 1e12,
                 "bwd_tflops": paper_flops(cl, ("bwd",)) / (bms / 1e3) / 1e12,
                 "fwd_ms": fms, "bwd_ms": bms, "per_rank": True}

    pk, pk_src = peaks()
    peak_burst = pk["bf16_tflops"]
    peak_sust = pk.get("bf16_tflops_sustained", peak_burst)
    mma_tflops = mma_flops_step * args.steps / (ms / 1e3) / 1e12

    # ---------------- roofline of the dominant kernel (rank 0's live CUDA-event timing) ----------------
    roof = None
    if prof:
        dom = max(prof, key=lambda n: prof[n][0])
        tot_ms, cnt = prof[dom]
        avg_ms = tot_ms / cnt
        w = kernel_work(dom, cl, out_bytes)
        step_share = tot_ms / ms if ms > 0 else None
        if w is not None:
            bound, amount = w  # algorithmic work of this rank's problem per step
            per_launch = amount * args.steps / cnt
            if bound == "tensor":
                # burst peak: the timed region is short (< 2 s at c3) and runs near the max SM clock
                # (clocks below); the sustained figure was measured at a 1335 MHz power-capped clock
                ach, unit, peak = per_launch / (avg_ms / 1e3) / 1e12, "TFLOP/s", peak_burst
            elif bound == "hbm":
                ach, unit, peak = per_launch / (avg_ms / 1e3) / 1e9, "GB/s", pk["hbm_gbs"]
            else:
                ach, unit = per_launch / (avg_ms / 1e3) / 1e12, "TFLOP/s"
                peak = alu_peak_tflops(clk.get("sm_max_mhz") or 1965.0)
            traffic, traffic_src = kernel_traffic(dom, c) if scaling == "weak" else (None, "not captured")
            roof = {"bound": bound, "kernel": dom, "achieved": ach, "peak": peak, "unit": unit,
                    "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                    "algorithmic_per_launch": per_launch, "avg_launch_ms": avg_ms, "launches": cnt,
                    "share_of_step": step_share,
                    "peak_source": (f"{pk_src} MEASURED_PEAKS.json bf16_tflops (burst)" if bound == "tensor"
                                    else f"{pk_src} hbm_gbs" if bound == "hbm"
                                    else "148 SM x 128 FP32 lanes x 2 x max SM clock")}
            if bound == "tensor":
                roof["frac_vs_sustained"] = ach / peak_sust
        roof_kernels = {n: {"ms_total": v[0], "launches": v[1]} for n, v in prof.items()}
    else:
        roof_kernels = {}

    # ---------------- end-to-end through the C ABI from pinned host buffers ----------------
    e2e = None
    if not args.no_e2e and c["bwd"] and args.mode == "bh":
        h_in = {n: x.pin_memory() for n, x in inp.items()}
        od = torch.float32 if args.out_f32 else torch.bfloat16
        h_out = {n: torch.empty(inp["q" if n in ("o", "dq") else "k"].shape, dtype=od).pin_memory()
                 for n in ("o", "dq", "dk", "dv", "dk2", "dv2")}
        h_out["lse"] = torch.empty((B, H, N), dtype=torch.float32).pin_memory()
        scratch = sa.host_step(h_in, h_out, w1, w2, det=det, out_f32=args.out_f32, device=dev)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        n_e2e = max(1, min(args.steps, 5))
        for _ in range(n_e2e):
            sa.host_step(h_in, h_out, w1, w2, det=det, out_f32=args.out_f32, scratch=scratch, device=dev)
        a1.record(stream)
        torch.cuda.synchronize()
        ems = a0.elapsed_time(a1)
        if dist:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": flops_step * n_e2e / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": sum(x.numel() * x.element_size() for x in h_in.values()) * world,
               "d2h_bytes_per_step": sum(x.numel() * x.element_size() for x in h_out.values()) * world,
               "ms_per_step": ems / n_e2e, "api": "simplicial_attn_host_step (pinned host buffers)"}
        del scratch

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(c)
        except Exception as ex:  # the baseline must never break the bench line
            cpu = {"value": None, "unit": "TFLOP/s", "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        fwd_path = sa.fwd_path(B, H, N, D, w1, w2, det=det, out_f32=args.out_f32)
        bwd_path = sa.bwd_path(B, H, N, D, w1, w2, det=det, out_f32=args.out_f32)
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None,
            "dtype": "bf16", "compute": "bf16 inputs; fp16 MMA operands, fp32 accumulate (tcgen05) / fp32 (SIMT)",
            "data": "synthetic",
            "config": dict(config_block(c, world, args.mode, scaling), shard_rank0=shard_desc),
            "mma_basis_tflops": mma_tflops,
            "pct_bf16_peak_mma_basis": 100.0 * mma_tflops / (peak_burst * world),
            "paths": {"fwd": {1: "simt", 2: "tcgen05"}.get(fwd_path, fwd_path),
                      "bwd": {1: "simt", 2: "tcgen05"}.get(bwd_path, bwd_path)},
            **extra,
            "roofline": roof, "kernels": roof_kernels,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "peaks": {"bf16_tflops": peak_burst, "bf16_tflops_sustained": peak_sust,
                      "hbm_gbs": pk["hbm_gbs"], "source": pk_src},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
