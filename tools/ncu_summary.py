"""Summarise an ncu report: key throughput metrics, instruction mix and top stall lines."""
import collections, csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))

def source(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]]

def main(rep, top=20):
    data, units = raw(rep)
    d = data[0]
    print(f"== {rep}: {d.get('Kernel Name', '')[:100]}")
    for k in KEYS:
        for kk in d:
            if kk == k or kk.endswith("." + k):
                print(f"  {k:80s} {d[kk]} {units.get(kk, '')}")
                break
    src = source(rep)
    ops = collections.Counter(); stall = collections.Counter(); tot = 0
    for r in src:
        s = r["Source"].strip()
        if not s:
            continue
        toks = s.split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        n = int(r["Instructions Executed"] or 0)
        ops[op.split(".")[0]] += n
        stall[op.split(".")[0]] += int(r["Warp Stall Sampling (All Samples)"] or 0)
        tot += n
    print(f"  total warp instructions {tot:.3e}")
    for op, n in ops.most_common(16):
        print(f"    {op:10s} {n:12d} {100 * n / max(tot, 1):5.1f}%  stall {stall[op]}")
    print("  top stall lines:")
    for r in sorted(src, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]:
        print(f"    {r['Warp Stall Sampling (All Samples)']:>7s} {r['Instructions Executed']:>10s}  {r['Source'][:90]}")

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)


def stall_lines(rep, reason="stall_long_sb", top=15, ctx=3):
    """Top SASS lines for one stall reason, with a few preceding instructions for context."""
    src = source(rep)
    idx = sorted(range(len(src)), key=lambda i: -int(src[i].get(reason) or 0))[:top]
    for i in sorted(idx):
        print(f"--- {src[i].get(reason)} samples")
        for j in range(max(0, i - ctx), i + 1):
            print(f"    {src[j].get(reason, ''):>7s} {src[j]['Instructions Executed']:>10s}  {src[j]['Source'][:100]}")


def cuda_lines(rep, top=25, reason=None):
    """Stall samples per CUDA source line (needs -lineinfo)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    res = []
    fname = None
    i = 0
    while i < len(lines):
        if lines[i].startswith('"File Name"'):
            fname = lines[i].split(",", 1)[1].strip('"').split("/")[-1]
            hdr = next(csv.reader([lines[i + 1]]))
            i += 2
            continue
        row = next(csv.reader([lines[i]]))
        if fname and len(row) == len(hdr):
            d = dict(zip(hdr, row))
            key = reason or "Warp Stall Sampling (All Samples)"
            try:
                n = int(d.get(key) or 0)
            except ValueError:
                n = 0
            if n:
                res.append((n, fname, d.get("Line No", d.get("#", "")), d.get("Source", "")[:110]))
        i += 1
    tot = sum(r[0] for r in res)
    for n, f, ln, s in sorted(res, reverse=True)[:top]:
        print(f"  {100 * n / tot:5.1f}% {f}:{ln}  {s.strip()}")


def _line_map(cubin, func_substr):
    """offset -> 'file:line' for the function whose mangled name contains func_substr (nvdisasm -g)."""
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur_fn, loc, mp = None, "?", {}
    import re
    for ln in out.splitlines():
        if ln.startswith(".text."):
            cur_fn = ln[6:].rstrip(":")
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and func_substr in cur_fn:
            mp[int(m.group(1), 16)] = loc
    return mp


def by_line(rep, cubin, func_substr, top=30, reason="Warp Stall Sampling (All Samples)"):
    mp = _line_map(cubin, func_substr)
    src = source(rep)
    base = int(src[0]["Address"], 16)
    agg, inst = collections.Counter(), collections.Counter()
    for r in src:
        off = int(r["Address"], 16) - base
        loc = mp.get(off, "?")
        agg[loc] += int(r.get(reason) or 0)
        inst[loc] += int(r["Instructions Executed"] or 0)
    tot = sum(agg.values())
    for loc, n in agg.most_common(top):
        print(f"  {100 * n / max(tot, 1):5.1f}%  {loc:24s} inst {inst[loc]:.3e}")
