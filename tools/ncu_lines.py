"""Warp-stall samples per CUDA source line of an ncu report (development tool).

    python tools/ncu_lines.py report.ncu-rep [N]

Runs `ncu -i report --page source --csv --print-source sass,cuda` and aggregates the sampled
stalls per (file, line), printing the top N lines with their two largest stall reasons.
"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    fname, hdr, rows = None, None, []
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("Function Name",) or r[0] == "":
            continue
        if len(r) != len(hdr) or r[2] != "-":
            continue
        try:
            float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        rows.append((fname, r))
    iall = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    tot = sum(float(r[iall] or 0) for _, r in rows)
    print("total samples", tot)
    for f, r in sorted(rows, key=lambda fr: -float(fr[1][iall] or 0))[:n]:
        s = float(r[iall] or 0)
        st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        sts = " ".join(f"{k}:{v / tot * 100:.1f}" for v, k in st if v > 0)
        print(f"{s / tot * 100:5.1f}% {f}:{r[0]:<5s} {r[1].strip()[:70]:70s} {sts}")


if __name__ == "__main__":
    main()
