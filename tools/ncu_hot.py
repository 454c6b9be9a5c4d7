"""Top SASS lines of an ncu report by warp-stall samples (development tool).

    ncu -i rep --page source --csv --print-source sass > src.csv; python tools/ncu_hot.py src.csv [N]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = rows[1]
    ia, isrc, iall, inot = (hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"),
                            hdr.index("Warp Stall Sampling (Not-issued Samples)"))
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(float(r[iall] or 0) for r in body)
    print("total samples", tot)
    for r in sorted(body, key=lambda r: -float(r[iall] or 0))[:n]:
        print(f"{r[ia]:>6s} {float(r[iall] or 0) / tot * 100:5.1f}% {float(r[inot] or 0) / tot * 100:5.1f}%  {r[isrc][:90]}")


if __name__ == "__main__":
    main()
