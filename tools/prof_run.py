"""Minimal launch sequence for ncu / compute-sanitizer (development tool).

    python tools/prof_run.py --config c4 --algo two_pass --iters 4

Generates the config's input, then launches the chosen entry point `iters` times on the
current stream (no flush), synchronising at the end.  Exits non-zero on any error.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

ALGO = {"two_pass": tp.ALGO_TWO_PASS, "recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--algo", default="two_pass")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--no-tma", action="store_true")
    ap.add_argument("--lookahead", type=int, default=0)
    ap.add_argument("--schedule", type=int, default=0)
    ap.add_argument("--cluster-size", type=int, default=0)
    args = ap.parse_args()
    x = workloads.generate(args.config, nrows=args.rows)
    if x.dtype == np.uint16:
        xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
    else:
        xd = torch.from_numpy(x).cuda()
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    for _ in range(args.iters):
        tp.softmax_ex(xd, ALGO[args.algo], out=y, disable_tma=args.no_tma, lookahead_rows=args.lookahead,
                      schedule=args.schedule, cluster_size=args.cluster_size)
    torch.cuda.synchronize()
    assert tp.watchdog_flags() == 0
    assert bool(torch.isfinite(y).all())
    print("ok", args.config, args.algo, tuple(xd.shape), tp.last_plan())


if __name__ == "__main__":
    main()
