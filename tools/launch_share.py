"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum ... --csv --log-file).

    python tools/launch_share.py profiles/r01_launches_bench_c4.csv
"""
import collections
import csv
import sys


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        # one line per kernel and grid: e.g. the cluster launch and its concurrent side launch
        per[int(r[ii])]["k"] = r[ki].split("(")[0][:60] + (f" grid={r[gi].strip('()').split(',')[0]}" if gi is not None else "")
    tot, cnt, by = collections.Counter(), collections.Counter(), collections.Counter()
    for d in per.values():
        k = d["k"]
        tot[k] += d.get("gpu__time_duration.sum", 0)
        cnt[k] += 1
        by[k] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    T = sum(tot.values())
    for k, t in tot.most_common():
        print(f"{k:72s} n={cnt[k]:4d} share={t / T:6.1%} mean_us={t / cnt[k] / 1e3:9.1f} "
              f"dram_MB_per_launch={by[k] / cnt[k] / 1e6:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
