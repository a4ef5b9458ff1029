"""Per-CUDA-source-line counters of an ncu report (ncu --page source --print-source
cuda,sass aggregates every SASS instruction onto its source line), top lines by
instructions executed and by warp-stall samples.

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fpath, hdr, lines = "", None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fpath = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit():
            d = dict(zip(hdr[4:], r[4:]))

            def f(k):
                try:
                    return float(d.get(k, "0"))
                except ValueError:
                    return 0.0

            lines.append((f"{fpath}:{r[0]}", r[1].strip()[:100], f("Instructions Executed"),
                          f("Warp Stall Sampling (All Samples)")))
    ti = sum(x[2] for x in lines) or 1
    ts = sum(x[3] for x in lines) or 1
    print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
    print("-- by instructions executed")
    for loc, s, i, st in sorted(lines, key=lambda x: -x[2])[:n]:
        print(f"{100 * i / ti:6.2f}% inst {100 * st / ts:6.2f}% stall  {loc:24s} {s}")
    print("-- by stall samples")
    for loc, s, i, st in sorted(lines, key=lambda x: -x[3])[:n]:
        print(f"{100 * i / ti:6.2f}% inst {100 * st / ts:6.2f}% stall  {loc:24s} {s}")


if __name__ == "__main__":
    main()
