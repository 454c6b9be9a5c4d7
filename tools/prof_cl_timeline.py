"""Per-row timeline of the cluster kernel (development tool).

    python tools/prof_cl_timeline.py c4b [--cluster-size 0] [--json out.json]

Runs one profiled launch of the Two-Pass cluster schedule (tp_set_profile_buffer) and prints, per
row iteration k, the median over CTAs (microseconds from the launch's first stamp) of: producer A's
first load of the row, team A's first and last pass-1 block, the tree warp's last local block value,
the row statistics, team B's first pass-2 command, the statistics seen by team B, team B's last
block — and the derived waits (tp_rowcl.cu ClTl).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

ROWS, SLOTS = 16, ["loadA", "A0", "A1", "tree", "stats", "B0", "Bstats", "B1"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--cluster-size", type=int, default=0)
    ap.add_argument("--json")
    args = ap.parse_args()
    x = workloads.generate(args.config)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else \
        torch.from_numpy(x).cuda()
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    for _ in range(3):
        tp.softmax_ex(xd, out=y, schedule=tp.SCHED_CLUSTER, cluster_size=args.cluster_size)
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(16 + ctas * ROWS * 8, dtype=torch.int64, device="cuda")
    tp.lib().tp_set_profile_buffer(buf.data_ptr())
    tp.softmax_ex(xd, out=y, schedule=tp.SCHED_CLUSTER, cluster_size=args.cluster_size)
    torch.cuda.synchronize()
    tp.lib().tp_set_profile_buffer(None)
    plan = tp.last_plan()
    t = buf[16:].cpu().numpy().reshape(ctas, ROWS, 8).astype(np.float64)
    t = t[: plan["grid_ctas"]]
    t0 = t[t > 0].min()
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)
    rows = []
    for k in range(ROWS):
        m = {s: float(np.nanmedian(t[:, k, i])) if np.isfinite(t[:, k, i]).any() else None
             for i, s in enumerate(SLOTS)}
        if m["A0"] is None:
            break
        d = t[:, k, :]
        der = {"A_dur": np.nanmedian(d[:, 2] - d[:, 1]), "tree_lag": np.nanmedian(d[:, 3] - d[:, 2]),
               "exchange": np.nanmedian(d[:, 4] - d[:, 3]), "B_stats_wait": np.nanmedian(d[:, 6] - d[:, 5]),
               "B_dur": np.nanmedian(d[:, 7] - d[:, 6]), "A_first_wait": np.nanmedian(d[:, 1] - d[:, 0]),
               "stats_spread": np.nanmax(d[:, 4]) - np.nanmin(d[:, 4])}
        rows.append({"k": k, **{s: round(v, 2) if v is not None else None for s, v in m.items()},
                     **{s: round(float(v), 2) for s, v in der.items()}})
    end = float(np.nanmax(t))
    out = {"config": args.config, "plan": plan, "end_us": round(end, 1), "rows": rows}
    for r in rows:
        print(" ".join(f"{k}={v}" for k, v in r.items()))
    print(json.dumps({"config": args.config, "plan": plan, "end_us": round(end, 1)}))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
