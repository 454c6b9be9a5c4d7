"""Cache-regime size sweep and SM-count scaling (the paper's F1/F2/F5/F6 size
sweeps and F8/F9 thread scaling).

    python tools/size_sweep.py [--json out.json]

1. Single rows of N = 2^10 .. 2^30 fp32 elements: Two-Pass vs Three-Pass (Recompute, Reload),
   under two cache protocols: "cold" (512 MB write + read before every rep: L2 holds clean,
   unrelated lines) and "warm" (no flush:
   input and output stay in L2 while they fit - the GPU analogue of PAPER.md:228's protocol,
   whose output eviction has no direct GPU counterpart since writes allocate in L2 too).
2. SM-count scaling: C4 (256 x 800,000 fp32) with the persistent grid capped at 1..148 CTAs
   (stream schedule) - the B200 analogue of the paper's thread scaling.
GB/s use each algorithm's compulsory bytes (12 / 16 / 20 B per element).
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

ALGOS = [("two_pass", tp.ALGO_TWO_PASS, 12), ("recompute", tp.ALGO_RECOMPUTE, 16), ("reload", tp.ALGO_RELOAD, 20)]


def timed(fn, pre, reps):
    for _ in range(2):
        pre()
        fn()
    ts = []
    for _ in range(reps):
        pre()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return float(np.median(ts))


def graph_us(fn, k=20):
    """Device time per launch of fn from a CUDA graph of k back-to-back launches (no host gaps;
    warm caches): the launch-latency-free figure for small sizes."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(k):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / (5 * k)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--max-log2", type=int, default=30)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    f32 = flush.view(torch.float32)

    def clean_flush():  # write 512 MB, then read it: L2 left holding clean lines only
        flush.zero_()
        tp.lib().tp_stream_baseline(4, f32.data_ptr(), f32.data_ptr(), f32.numel(), 1.0, 0, tp._stream())

    out = {"size_sweep": [], "sm_scaling": []}
    for lg in range(10, args.max_log2 + 1):
        n = 1 << lg
        x = torch.from_numpy(workloads.uniform(n, -100.0, 100.0, seed=lg, stream=30)).cuda().reshape(1, n)
        y = torch.empty_like(x)
        reps = 25 if n <= (1 << 24) else 7
        for name, algo, bpe in ALGOS:
            fn = (lambda a=algo: tp.softmax_ex(x, a, out=y))
            t_cold = timed(fn, clean_flush, reps)
            t_warm = timed(fn, lambda: None, reps)
            rec = {"n": n, "algo": name, "cold_us": t_cold * 1e6, "cold_GBps": bpe * n / t_cold / 1e9,
                   "warm_us": t_warm * 1e6, "warm_GBps": bpe * n / t_warm / 1e9}
            if n <= (1 << 24):
                tg = graph_us(fn)
                rec.update(graph_us=tg, graph_GBps=bpe * n / (tg * 1e-6) / 1e9)
            out["size_sweep"].append(rec)
            print(json.dumps(rec), flush=True)
        del x, y
        torch.cuda.empty_cache()
    x = torch.from_numpy(workloads.generate("c4")).cuda()
    y = torch.empty_like(x)
    for g in (1, 2, 4, 8, 16, 32, 64, 96, 128, 148):
        t = timed(lambda: tp.softmax_ex(x, out=y, grid_ctas=g, schedule=tp.SCHED_STREAM), clean_flush, 5)
        rec = {"ctas": g, "us": t * 1e6, "GBps": 12 * x.numel() / t / 1e9}
        out["sm_scaling"].append(rec)
        print(json.dumps(rec), flush=True)
    assert tp.watchdog_flags() == 0
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
