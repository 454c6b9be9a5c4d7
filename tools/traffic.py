"""DRAM traffic per call of each workload's dominant kernel(s) from ncu launch lists (measurement).

    python tools/traffic.py <tag> [--dir gpurun_out] [--out profiles/traffic.json]

Reads <dir>/<tag>_traffic_<cfg>.csv, each an ncu launch list (dram__bytes_read.sum,
dram__bytes_write.sum, gpu__time_duration.sum) of `tools/prof_run.py --config <cfg> --iters 4`
captured with --cache-control none: consecutive calls, so a call's bytes include the write-back
of the previous call's dirty L2 lines, which a flushed single capture misses.  Calls 2..4 are
averaged (call 1 starts from a cold L2).  A call is every launch of the library's kernels between
two calls (a cluster launch and its concurrent side launch count together).
"""
import argparse
import csv
import io
import json
import os
import sys

OURS = ("stream_kernel", "rowcl_kernel", "rowph_kernel", "small_kernel", "general_kernel", "rowres_kernel")
KNAME = {"c5": "tp::rowph_kernel<float,kTwoPass>", "c3": "tp::stream_kernel<float,kTwoPass>",
         "c4": "tp::rowcl_kernel<float>", "c4b": "tp::rowres_kernel<uint16_t>", "c2": "tp::small_kernel<float>"}
ALG = {"c5": 12 * 2 ** 31, "c3": 12 * 2 ** 26, "c4": 12 * 256 * 800000, "c4b": 8 * 256 * 800000,
       "c2": 12 * 64 * 32768}


def launches(path):
    txt = open(path, errors="replace").read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    out = {}
    for r in rows:
        d = out.setdefault(int(r["ID"]), {"name": r["Kernel Name"], "grid": r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return [out[k] for k in sorted(out)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--dir", default="gpurun_out")
    ap.add_argument("--out", default="profiles/traffic.json")
    args = ap.parse_args()
    res = {"_about": __doc__.strip().splitlines()[0] + " Source: " + args.tag + " (tools/traffic.py)."}
    for cfg in KNAME:
        p = os.path.join(args.dir, f"{args.tag}_traffic_{cfg}.csv")
        if not os.path.exists(p):
            continue
        ls = [l for l in launches(p) if any(k in l["name"] for k in OURS)]
        # group into calls: prof_run issues 4 calls; a call = its main launch (+ the side launch
        # of a split cluster call, which has a smaller grid and follows it)
        calls, cur = [], None
        main_name = None
        for l in ls:
            if cur is None or (l["name"] == main_name and l["grid"] == cur[0]["grid"]):
                cur = [l]
                calls.append(cur)
                main_name = l["name"]
            else:
                cur.append(l)
        use = calls[1:] if len(calls) > 1 else calls
        rd = sum(sum(l["dram__bytes_read.sum"] for l in c) for c in use) / len(use)
        wr = sum(sum(l["dram__bytes_write.sum"] for l in c) for c in use) / len(use)
        us = sum(sum(l["gpu__time_duration.sum"] for l in c) for c in use) / len(use) / 1e3
        res[cfg] = {"kernel": KNAME[cfg], "launches_per_call": len(use[0]), "calls_averaged": len(use),
                    "read": round(rd), "write": round(wr), "dram_bytes_per_launch": round(rd + wr),
                    "algorithmic_bytes": ALG[cfg], "dram_over_algorithmic": round((rd + wr) / ALG[cfg], 4),
                    "duration_us_under_ncu": round(us, 2), "source": os.path.basename(p)}
    json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
