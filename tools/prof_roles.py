"""Per-role cycle breakdown of the cluster kernel (development tool).

    python tools/prof_roles.py c4 [--reps 5] [--cluster-size 0]

Installs a counter buffer (tp_set_profile_buffer), runs the Two-Pass cluster schedule, and prints
where compute warp 0 and the producer of an average CTA spend their clock cycles.
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

SLOTS = ["cmd_wait", "full_wait", "row_wait_and_stats", "p1_compute", "p2_compute", "teamA_total",
         "prod_free_stage_wait", "prod_push_wait", "prod_total", "ctas", "teamB_total", "teamB_full_wait",
         "teamB_cmd_wait"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cluster-size", type=int, default=0)
    args = ap.parse_args()
    x = workloads.generate(args.config)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else \
        torch.from_numpy(x).cuda()
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    tp.softmax_ex(xd, out=y, schedule=tp.SCHED_CLUSTER, cluster_size=args.cluster_size)
    buf = torch.zeros(16, dtype=torch.int64, device="cuda")
    tp.lib().tp_set_profile_buffer(buf.data_ptr())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.reps):
        tp.softmax_ex(xd, out=y, schedule=tp.SCHED_CLUSTER, cluster_size=args.cluster_size)
    e.record()
    e.synchronize()
    tp.lib().tp_set_profile_buffer(None)
    c = buf.cpu().numpy().astype(np.float64)
    ctas = c[9]
    per = {SLOTS[i]: c[i] / ctas for i in range(13) if i != 9}
    tot = per["teamA_total"] + per["teamB_total"]
    out = {"config": args.config, "plan": tp.last_plan(), "us_per_launch": s.elapsed_time(e) * 1e3 / args.reps,
           "cycles_per_cta": {k: round(v) for k, v in per.items()},
           "share_of_both_teams": {k: round(per[k] / tot, 3) for k in SLOTS[:5]},
           "producer_share": {k: round(per[k] / per["prod_total"], 3) for k in SLOTS[6:8]}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
