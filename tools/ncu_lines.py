"""Per-CUDA-source-line warp stall samples of an ncu report (needs -lineinfo + --import-source).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv, io, subprocess, sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    path, hdr, rows = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        try:
            samples = int(r[4])
            nis = int(r[5])
            inst = int(r[7])
        except (ValueError, IndexError):
            continue
        rows.append((samples, nis, inst, f"{path}:{r[0]}", r[1].strip()[:90]))
    tot = sum(x[0] for x in rows) or 1
    rows.sort(reverse=True)
    print(f"total stall samples {tot}")
    for s, n, i, loc, src in rows[:top]:
        print(f"{100 * s / tot:6.2f}% {s:8d} {n:7d} {i:11d}  {loc:22s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
