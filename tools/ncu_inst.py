"""Executed instructions per CUDA source line and per SASS opcode of an ncu report (development tool).

    python tools/ncu_inst.py report.ncu-rep [N]
"""
import collections
import csv
import io
import os
import subprocess
import sys


def rows(rep, what):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", what],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(txt)))


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    # per opcode (SASS view)
    r = rows(rep, "sass")
    hdr = next(x for x in r if x and x[0] == "Address")
    ii, si = hdr.index("Instructions Executed"), hdr.index("Source")
    ops = collections.Counter()
    tot = 0
    for x in r:
        if len(x) != len(hdr) or x[0] == "Address":
            continue
        try:
            v = float(x[ii] or 0)
        except ValueError:
            continue
        op = x[si].split()
        op = [t for t in op if not t.startswith("@")]
        ops[op[0].split(".")[0] if op else "?"] += v
        tot += v
    print(f"warp instructions executed: {tot:.0f}")
    for k, v in ops.most_common(25):
        print(f"  {k:12s} {v / tot * 100:5.1f}%  {v:.0f}")
    # per CUDA line (sass,cuda view: CUDA rows carry the aggregated metrics)
    r = rows(rep, "sass,cuda")
    fname, hdr, per = None, None, []
    for x in r:
        if not x:
            continue
        if x[0] == "File Path":
            fname = os.path.basename(x[1])
            continue
        if x[0] == "Line No":
            hdr = x
            continue
        if hdr is None or len(x) != len(hdr) or x[2] != "-":
            continue
        try:
            v = float(x[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        per.append((v, fname, x[0], x[1].strip()[:80]))
    per.sort(reverse=True)
    print("top lines by executed warp instructions:")
    for v, f, ln, src in per[:n]:
        print(f"  {v / tot * 100:5.1f}% {f}:{ln:<5s} {src}")


if __name__ == "__main__":
    main()
