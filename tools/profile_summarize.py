"""Summarise the round's ncu captures (tools/profile_round.sh) into profiles/:
  profiles/<tag>_launches_c3.csv      per-launch gpu__time_duration of one bench step (cold, serialised)
  profiles/<tag>_ncu_<kernel>.txt     key metrics, instruction mix, top stall lines (tools/ncu_summary.py)
  profiles/<tag>_traffic_c3.json      per-kernel DRAM bytes per launch (dram__bytes_read+write), the
                                      `traffic` bench.py reports for the dominant kernel
usage: python tools/profile_summarize.py <tag>"""
import csv, io, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("SA_PROF_DIR", os.path.join(ROOT, "profiles"))


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return dict(zip(hdr, rows[2])), dict(zip(hdr, units))


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(tag, prefix="", cfg="c3"):
    traffic = {}
    for k in ("tc_fwd", "tc_bwd_q", "tc_bwd_kv"):
        rep = os.path.join(OUT, f"{prefix}full_{k}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d, u = raw_metrics(rep)
        rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        t_ns = float(d["gpu__time_duration.sum"].replace(",", "")) * {"ns": 1, "us": 1e3, "ms": 1e6}.get(
            u["gpu__time_duration.sum"], 1)
        traffic[k] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                      "ncu_duration_ms": t_ns / 1e6,
                      "tensor_pipe_pct": next((float(v) for kk, v in d.items() if kk.endswith(
                          "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")), None),
                      "report": f"gpurun_out/{prefix}full_{k}.ncu-rep (not committed; summary in {tag}_{prefix}ncu_{k}.txt)"}
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                             capture_output=True, text=True).stdout
        lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "30"],
                               capture_output=True, text=True).stdout
        with open(os.path.join(PROF, f"{tag}_{prefix}ncu_{k}.txt"), "w") as f:
            f.write(txt + "\n== per-CUDA-line warp stall samples (tools/ncu_lines.py)\n" + lines)
    if not traffic:
        return
    with open(os.path.join(PROF, f"{tag}_traffic_{cfg}.json"), "w") as f:
        json.dump({"config": cfg, "capture": "ncu --set full --clock-control none, one launch each, bench.py "
                   + ("--sweep membound" if prefix else "") + " --steps 1 --warmup 1", "kernels": traffic}, f, indent=1)
    src = os.path.join(OUT, "launches_c3.csv")
    if not prefix and os.path.exists(src):
        shutil.copy(src, os.path.join(PROF, f"{tag}_launches_c3.csv"))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    main(tag)
    main(tag, prefix="mb_", cfg="membound")
