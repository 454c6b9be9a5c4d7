"""Per-rank work of the sharded configurations, measured on one GPU (measurement tool).

    python tools/shard_projection.py [--reps 10] [--out profiles/r02d_shard_projection.json]

`bench.py --gpus N` runs the sharded paths on N GPUs; a gpurun call has one GPU, so this tool
times what ONE rank of an N-rank job computes, on the one GPU, with no other rank involved (no
waiting between ranks, no exchange):

  C5 chunk-sharded (north_star): rank 0's chunk of 2^31 / N elements of the C5 row, the partial
      launch (pass 1 of the chunk) then the finish launch (pass 2 of the chunk, given N pairs),
      back to back with CUDA events on the launching stream.  The 8-byte-per-rank all-gather
      between them (NCCL over NVLink / NVSwitch) is NOT included: it is not measurable on one GPU.
  C4 rows-sharded: rank 0's 256 / N rows, one softmax call (no exchange exists).

Projected aggregate = N x the rank's algorithmic bytes / its time: an upper bound for the N-GPU
job (exchange latency and rank skew come on top), reported as such, never as a bench value.
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


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) * 1e3 for a, b in ev]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out")
    args = ap.parse_args()
    res = {"about": __doc__.strip().splitlines()[0], "c5_chunk": [], "c4_rows": []}
    n5 = 1 << 31
    for w in (1, 2, 4, 8):
        n = n5 // w
        x = torch.from_numpy(workloads.generate("c5", col0=0, ncols=n)).cuda()
        y = torch.empty_like(x)
        ws = tp.new_workspace(1, n)
        pr = tp.partial(x, workspace=ws)
        pairs = pr.view(1, 1, 2).repeat(w, 1, 1).contiguous()  # timing only: the rank's pair N times
        t_p = timed(lambda: tp.partial(x, out=pr, workspace=ws), args.reps)
        plan_p = tp.last_plan()
        t_f = timed(lambda: tp.finish(x, pairs, w, out=y, workspace=ws), args.reps)
        plan_f = tp.last_plan()

        def step():
            tp.partial(x, out=pr, workspace=ws)
            tp.finish(x, pairs, w, out=y, workspace=ws)

        t_s = timed(step, args.reps)
        gbs = 12.0 * n / (t_s * 1e-6) / 1e9
        res["c5_chunk"].append({"world": w, "chunk_elements": n, "partial_us": round(t_p, 1), "finish_us": round(t_f, 1),
                                "rank_step_us": round(t_s, 1), "rank_GBps": round(gbs, 1),
                                "projected_aggregate_GBps_upper_bound": round(w * gbs, 1),
                                "plans": [plan_p, plan_f]})
        print(json.dumps(res["c5_chunk"][-1]), flush=True)
        del x, y, ws
        torch.cuda.empty_cache()
    for w in (1, 2, 4, 8):
        r = 256 // w
        x = torch.from_numpy(workloads.generate("c4", row0=0, nrows=r)).cuda()
        y = torch.empty_like(x)
        t = timed(lambda: tp.softmax(x, out=y), args.reps)
        gbs = 12.0 * x.numel() / (t * 1e-6) / 1e9
        res["c4_rows"].append({"world": w, "rows": r, "us": round(t, 1), "rank_GBps": round(gbs, 1),
                               "projected_aggregate_GBps": round(w * gbs, 1), "plan": tp.last_plan()})
        print(json.dumps(res["c4_rows"][-1]), flush=True)
        del x, y
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
