"""Quick per-config timing of the library kernels (development tool; bench.py is the contract).

For each config: warm-up, then 25 reps, each preceded by an L2 flush, timed with CUDA events
on the launching stream; prints median GB/s against the paper's cost model (12/16/20 B per
fp32 element; 8/10/16 for bf16 in).
"""
import argparse
import json
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

BYTES = {("two_pass", "f32"): 12, ("recompute", "f32"): 16, ("reload", "f32"): 20,
         ("two_pass", "bf16"): 8, ("recompute", "bf16"): 10, ("reload", "bf16"): 16}
ALGO = {"two_pass": tp.ALGO_TWO_PASS, "recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c4,c4b")
    ap.add_argument("--algos", default="two_pass,recompute,reload")
    ap.add_argument("--reps", type=int, default=25)
    ap.add_argument("--flush", type=int, default=1)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = []
    for key in args.configs.split(","):
        cfg = workloads.CONFIGS[key]
        x = workloads.generate(key)
        if cfg.dtype == "bf16":
            xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
        else:
            xd = torch.from_numpy(x).cuda()
        del x
        y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
        for algo in args.algos.split(","):
            for _ in range(3):
                tp.softmax_ex(xd, ALGO[algo], out=y)
            ts = []
            for _ in range(args.reps):
                if args.flush:
                    flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                tp.softmax_ex(xd, ALGO[algo], out=y)
                e.record()
                e.synchronize()
                ts.append(s.elapsed_time(e) * 1e-3)
            t = float(np.median(ts))
            gbs = BYTES[(algo, cfg.dtype)] * cfg.elements / t / 1e9
            rec = dict(config=key, algo=algo, median_us=t * 1e6, min_us=min(ts) * 1e6, alg_GBps=gbs,
                       elems_per_s=cfg.elements / t, watchdog=tp.watchdog_flags())
            out.append(rec)
            print(json.dumps(rec), flush=True)
        del xd, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
