"""Randomised soak (development / robustness evidence): random shapes, dtypes, algorithms and
schedules; every result bitwise against the same algorithm on the stream schedule, the watchdog
clear, and small cases against the oracle.

    python tools/soak.py --minutes 10 [--seed 0]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402
from gpu_helpers import assert_parity  # noqa: E402

SCHEDS = [tp.SCHED_AUTO, tp.SCHED_CLUSTER, tp.SCHED_SMALL, tp.SCHED_HOLD, tp.SCHED_PHASE, tp.SCHED_RESIDENT]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=10.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--clamp-frac", type=float, default=0.1)
    ap.add_argument("--bf16-frac", type=float, default=0.3)
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + 60 * args.minutes
    n = bad = 0
    while time.time() < t_end:
        nb = int(rng.choice([1, 2, 3, 5, 17, 49, 64, 65, 130, 300]))
        cols = max(1, nb * 16384 - int(rng.integers(0, 16384)))
        rows = int(rng.integers(1, max(2, min(300, (64 << 20) // (cols * 4)))))
        dtype = "bf16" if rng.random() < args.bf16_frac else "f32"
        algo = int(rng.choice([tp.ALGO_TWO_PASS, tp.ALGO_RECOMPUTE, tp.ALGO_RELOAD]))
        sched = int(rng.choice(SCHEDS))
        cl = int(rng.choice([0, 1, 2, 4, 8]))
        if sched == tp.SCHED_RESIDENT:  # CTAs per row: automatic, one block each, or 2-3 blocks each
            cl = int(rng.choice([0, nb, -(-nb // 3), -(-nb // 2), -(-nb // 3) + 1]))
        grid = int(rng.choice([0, 0, 0, 7, 33]))
        x = workloads.ragged_case(rows, cols, -400.0, 400.0, seed=n, stream=7)
        if rng.random() < args.clamp_frac:  # out of domain: the clamped path, in a few rows
            for r in rng.integers(0, rows, 1 + rows // 8):
                x[int(r), int(rng.integers(0, cols))] = 3.0e7
        if dtype == "bf16":
            x = workloads.to_bf16(x)
            xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
        else:
            xd = torch.from_numpy(x).cuda()
        ref = tp.softmax_ex(xd, algo, schedule=tp.SCHED_STREAM)
        if algo == tp.ALGO_TWO_PASS and rng.random() < 0.15:  # the split path: partial / finish
            W = int(rng.choice([1, 2, 4]))
            per = -(-(-(-cols // 16384)) // W) * 16384  # block-aligned chunk width
            chunks = [xd[:, w * per:min(cols, (w + 1) * per)].contiguous() for w in range(W)]
            chunks = [c for c in chunks if c.shape[1]]
            pairs = torch.stack([tp.partial(c) for c in chunks])
            y = torch.cat([tp.finish(c, pairs, len(chunks)) for c in chunks], dim=1)
            plan = {"split": len(chunks)}
            same = bool(torch.equal(y, ref))
            if not same and (len(chunks) & (len(chunks) - 1)) == 0 and cols % (16384 * len(chunks)) == 0:
                bad += 1
                print(json.dumps({"bad_split": [rows, cols, dtype, W]}), flush=True)
            n += 1
            del x, xd, ref, y
            continue
        if algo == tp.ALGO_TWO_PASS and rng.random() < 0.05:  # the host-buffer pipeline
            hx = xd.cpu().pin_memory()
            hy = tp.softmax_host(hx)
            if not torch.equal(hy, tp.softmax_ex(xd, algo).cpu()):
                bad += 1
                print(json.dumps({"bad_host": [rows, cols, dtype]}), flush=True)
            n += 1
            del x, xd, ref, hx, hy
            continue
        y = tp.softmax_ex(xd, algo, schedule=sched, cluster_size=cl, grid_ctas=grid)
        plan = tp.last_plan()
        ok = bool(torch.equal(y, ref)) and tp.watchdog_flags() == 0
        if ok and rows * cols <= 2_000_000 and not (x == 3.0e7).any():
            try:
                assert_parity(x, y.cpu().numpy(), "soak")
            except AssertionError:
                ok = False
        n += 1
        if not ok:
            bad += 1
            print(json.dumps({"bad": [rows, cols, dtype, algo, sched, cl, grid], "plan": plan}), flush=True)
        del x, xd, ref, y
    print(json.dumps({"cases": n, "bad": bad}))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
