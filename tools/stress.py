"""Repeated launches with a watchdog check after each (development tool).

    python tools/stress.py c4:two_pass c4b:two_pass:schedule=2 --reps 50

For each spec: `reps` launches, each timed with CUDA events and followed by a synchronise, a
watchdog-flag read (reset on error) and a bitwise comparison with the first launch's output;
prints the time distribution and every failing launch.
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

ALGO = {"two_pass": tp.ALGO_TWO_PASS, "recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--flush", type=int, default=1)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    cache = {}
    for spec in args.specs:
        key, algo = spec.split(":")[:2]
        opts = {k: int(v) for k, v in (kv.split("=") for kv in spec.split(":")[2:])}
        if key not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            x = workloads.generate(key)
            cache[key] = (torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
                          if x.dtype == np.uint16 else torch.from_numpy(x).cuda())
        xd = cache[key]
        y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
        ts, bad, ref = [], [], None
        for i in range(args.reps):
            if args.flush:
                flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            tp.softmax_ex(xd, ALGO[algo], out=y, **opts)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
            f = tp.watchdog_flags()
            if ref is None:
                ref = y.clone()
            same = bool(torch.equal(y, ref))
            if f or not same:
                bad.append((i, f, same, ts[-1]))
        ts = np.array(ts)
        print(json.dumps(dict(spec=spec, median_us=float(np.median(ts)), min_us=float(ts.min()),
                              max_us=float(ts.max()), p90_us=float(np.percentile(ts, 90)), n_bad=len(bad), plan=tp.last_plan(),
                              bad=bad[:10])), flush=True)


if __name__ == "__main__":
    main()
