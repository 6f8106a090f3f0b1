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
