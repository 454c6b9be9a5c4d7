"""A/B of the resident-row schedule (tp_rowres.cu) against the cluster and stream schedules
(development tool): bitwise agreement, then back-to-back timing of each schedule on C4 / C4b
and a few forced group sizes.  Prints one JSON line per (config, schedule)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

BYTES = {"f32": 12, "bf16": 8}


def timed(fn, reps, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) * 1e3 / reps  # us per call


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c4b,c4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--groups", default="0")
    ap.add_argument("--only-resident", action="store_true")
    ap.add_argument("--ahead", default="0")
    ap.add_argument("--algo", default="two_pass", choices=["two_pass", "recompute", "reload"])
    args = ap.parse_args()
    algo = {"two_pass": tp.ALGO_TWO_PASS, "recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}[args.algo]
    for key in args.configs.split(","):
        cfg = workloads.CONFIGS[key]
        x = workloads.generate(key)
        if cfg.dtype == "bf16":
            xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
        else:
            xd = torch.from_numpy(x).cuda()
        del x
        y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
        ws = tp.new_workspace(*xd.shape)
        ref = None
        scheds = [] if args.only_resident else [("stream", tp.SCHED_STREAM, 0), ("cluster", tp.SCHED_CLUSTER, 0)]
        scheds = [(n, sc, g, 0) for n, sc, g in scheds]
        scheds += [(f"resident_g{g}_a{la}", tp.SCHED_RESIDENT, int(g), int(la)) for g in args.groups.split(",")
                   for la in args.ahead.split(",")]
        for name, sc, g, la in scheds:
            tp.softmax_ex(xd, algo, out=y, workspace=ws, schedule=sc, cluster_size=g, lookahead_rows=la)
            torch.cuda.synchronize()
            plan = tp.last_plan()
            h = y.cpu().numpy()
            if ref is None:
                ref = h.copy()
            same = bool(np.array_equal(ref, h))
            us = timed(lambda: tp.softmax_ex(xd, algo, out=y, workspace=ws, schedule=sc, cluster_size=g, lookahead_rows=la),
                       args.reps)
            gbs = BYTES[cfg.dtype] * cfg.elements / (us * 1e-6) / 1e9
            print(json.dumps(dict(config=key, algo=args.algo, sched=name, plan=plan, us=us, alg_GBps=gbs, bitwise_vs_stream=same,
                                  watchdog=tp.watchdog_flags(ws))), flush=True)


if __name__ == "__main__":
    main()
