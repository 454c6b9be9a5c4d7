"""Per-pass decomposition and STREAM-style baselines on B200 (PAPER.md:285-301,
323-329: every softmax pass is bandwidth-bound).

    python tools/pass_decomp.py [--configs c4,c3] [--reps 15] [--json out.json]

For each workload (fp32): STREAM copy / scale / in-place scale / read-only sum over the same
number of elements, Two-Pass pass 1 alone (softmax_partial_ex: read x, one (m, n) per row),
pass 2 alone (softmax_finish_ex with those pairs: read x, write y), the whole Two-Pass on the
default and on the stream schedule, the Three-Pass comparators, and every pass of every
algorithm alone on the stream kernel (tp_phase_only: the paper's per-pass runtime figure,
PAPER.md:323-329).  Every rep is preceded by
an L2 flush (512 MB write, then a 512 MB read so that no dirty line is left to write back
inside the timed region) and timed with CUDA events on the launching stream; medians.
GB/s use each kernel's own compulsory bytes (Table 2 l.180-198).
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


def clean_flush(flush):
    """Evict L2 and leave it holding CLEAN lines: a 512 MB write alone would leave ~126 MB of
    dirty lines whose write-back then lands inside the timed kernel."""
    flush.zero_()
    f = flush.view(torch.float32)
    tp.lib().tp_stream_baseline(4, f.data_ptr(), f.data_ptr(), f.numel(), 1.0, 0,
                                torch.cuda.current_stream().cuda_stream)


def timeit(fn, reps, flush):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        clean_flush(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c4,c3")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    L = tp.lib()
    stream = torch.cuda.current_stream().cuda_stream
    out = []
    for key in args.configs.split(","):
        x = torch.from_numpy(workloads.generate(key)).cuda()
        rows, cols = x.shape
        n = x.numel()
        y = torch.empty_like(x)
        tmp = torch.empty_like(x)
        part = torch.empty(4096, dtype=torch.float32, device="cuda")
        ws = tp.new_workspace(rows, cols)
        pairs = tp.partial(x, workspace=ws).reshape(1, rows, 2).contiguous()

        def sb(what, dst=None):
            return lambda: L.tp_stream_baseline(what, tmp.data_ptr() if what == 2 else x.data_ptr(),
                                                (part if what == 3 else y).data_ptr(), n, 1.0, 0, stream)
        cases = [
            ("stream_copy", sb(0), 8), ("stream_scale", sb(1), 8), ("stream_scale_inplace", sb(2), 8),
            ("stream_read_sum", sb(3), 4),
            ("two_pass_pass1_only", lambda: tp.partial(x, workspace=ws), 4),
            ("two_pass_pass2_only", lambda: tp.finish(x, pairs, 1, out=y), 8),
            ("two_pass", lambda: tp.softmax_ex(x, out=y, workspace=ws), 12),
            ("two_pass_stream_schedule", lambda: tp.softmax_ex(x, out=y, workspace=ws, schedule=tp.SCHED_STREAM), 12),
            ("three_pass_recompute", lambda: tp.softmax_ex(x, tp.ALGO_RECOMPUTE, out=y, workspace=ws), 16),
            ("three_pass_reload", lambda: tp.softmax_ex(x, tp.ALGO_RELOAD, out=y, workspace=ws), 20),
        ]
        # each pass of each algorithm alone (tp_phase_only, stream kernel; the statistics of the
        # later passes come from a full stream-schedule call on the same workspace first):
        # the paper's Fig. "absolute runtime of the passes"
        pws = {a: tp.new_workspace(rows, cols) for a in (tp.ALGO_TWO_PASS, tp.ALGO_RECOMPUTE, tp.ALGO_RELOAD)}
        ybuf = torch.empty_like(x)
        for a, pws_a in pws.items():
            tp.softmax_ex(x, a, out=ybuf, workspace=pws_a, schedule=tp.SCHED_STREAM)
        phase_bytes = {("two_pass", 0): 4, ("two_pass", 1): 8, ("recompute", 0): 4, ("recompute", 1): 4,
                       ("recompute", 2): 8, ("reload", 0): 4, ("reload", 1): 8, ("reload", 2): 8}
        anum = {"two_pass": tp.ALGO_TWO_PASS, "recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}
        for (an, ph), bpe in phase_bytes.items():
            cases.append((f"{an}_phase{ph + 1}_alone",
                          (lambda an=an, ph=ph: tp.phase_only(x, anum[an], ph, pws[anum[an]], out=ybuf)), bpe))
        for name, fn, bpe in cases:
            t = timeit(fn, args.reps, flush)
            rec = {"config": key, "kernel": name, "median_us": round(t * 1e6, 2), "bytes_per_elem": bpe,
                   "GBps": round(bpe * n / t / 1e9, 1), "elems_per_s": n / t}
            if name.startswith(("two_pass", "three", "recompute", "reload")):
                rec["plan"] = tp.last_plan()
            out.append(rec)
            print(json.dumps(rec), flush=True)
        del x, y, tmp, ws, pws, ybuf
        torch.cuda.empty_cache()
    assert tp.watchdog_flags() == 0
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
