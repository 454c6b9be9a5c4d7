"""Launch-parameter sweep (development tool): lookahead rows and grid size for one config.

    TP_L2_HINTS=0|1 python tools/sweep.py --config c4 --lookaheads 0,4,8,12,16 --grids 0
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

BYTES = {"f32": 12, "bf16": 8}
ALGO = {"two_pass": tp.ALGO_TWO_PASS, "recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--algo", default="two_pass")
    ap.add_argument("--lookaheads", default="0")
    ap.add_argument("--grids", default="0")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--schedule", type=int, default=0)
    args = ap.parse_args()
    cfg = workloads.CONFIGS[args.config]
    x = workloads.generate(args.config)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else \
        torch.from_numpy(x).cuda()
    del x
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for g in [int(v) for v in args.grids.split(",")]:
        for la in [int(v) for v in args.lookaheads.split(",")]:
            run = lambda: tp.softmax_ex(xd, ALGO[args.algo], out=y, grid_ctas=g, lookahead_rows=la,
                                                schedule=args.schedule)  # noqa: E731
            for _ in range(3):
                run()
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                run()
                e.record()
                e.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            t = float(np.median(ts))
            print(json.dumps({"config": args.config, "algo": args.algo, "grid": g, "lookahead": la,
                              "hints": os.environ.get("TP_L2_HINTS", "1"), "schedule": args.schedule, "median_us": round(t, 2),
                              "alg_GBps": round(BYTES[cfg.dtype] * cfg.elements / t / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
