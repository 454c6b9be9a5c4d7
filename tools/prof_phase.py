"""Per-role cycle breakdown of the phase kernel (development tool; tp_rowph.cu PhProf slots).

    python tools/prof_phase.py c3 [--reps 5]

Builds (once) and loads paper_2001_04438_b200/libtwopass_prof.so, compiled with -DTP_PH_PROF.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
_PROF_SO = os.environ.get("TP_PROF_LIBRARY") or os.path.join(ROOT, "paper_2001_04438_b200", "libtwopass_prof.so")
os.environ["TP_LIBRARY"] = _PROF_SO  # before the package import: the binding reads it then
from paper_2001_04438_b200 import build as _build  # noqa: E402
if not os.path.exists(_PROF_SO):
    _build.build(out=_PROF_SO, defines=("TP_PH_PROF",))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

SLOTS = ["p1_full_wait", "p1_slot_wait", "p1_work", "p2_stats_wait", "p2_full_wait", "p2_work",
         "tree_wait", "tree_work", "tree_retire", "tree_batches", "tree_blocks",
         "prod_empty_wait", "prod_total", "compute_total", "tree_total", "ctas"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warm", type=int, default=0, help="untimed calls first (sustained load, power cap)")
    args = ap.parse_args()
    x = workloads.generate(args.config)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else \
        torch.from_numpy(x).cuda()
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    tp.softmax_ex(xd, out=y, schedule=tp.SCHED_PHASE)
    for _ in range(args.warm):
        tp.softmax_ex(xd, out=y, schedule=tp.SCHED_PHASE)
    buf = torch.zeros(16 + 5 * 200 + 8, dtype=torch.int64, device="cuda")
    tp.lib().tp_set_profile_buffer(buf.data_ptr())
    buf.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.reps):
        tp.softmax_ex(xd, out=y, schedule=tp.SCHED_PHASE)
    e.record()
    e.synchronize()
    tp.lib().tp_set_profile_buffer(None)
    c = buf.cpu().numpy().astype(np.float64)
    rt = buf[16 + 5 * 200:16 + 5 * 200 + 2].cpu().numpy()  # the row tree's start / end (last launch)
    tl = buf[16:16 + 5 * 200].cpu().numpy().reshape(-1, 5)  # last launch's per-CTA timeline (ns)
    tl = tl[tl[:, 0] > 0]
    if not tl.size:
        print("no timeline (counters only)", c[:16].tolist())
        tl = np.zeros((1, 5), dtype=np.int64)
    t0 = tl[:, 0].min()
    rel = (tl - t0) / 1e3
    print("timeline us (min / median / max over CTAs): start, pass-1 end, stats seen, last retirement, end")
    for i, nm in enumerate(["start", "p1_end", "stats", "retired", "end"]):
        col = rel[:, i][tl[:, i] > 0]
        if col.size:
            print(f"  {nm:9s} {col.min():9.1f} {np.median(col):9.1f} {col.max():9.1f}")
    if rt[0] > 0:
        print(f"  row tree  {(rt[0] - t0) / 1e3:9.1f} .. {(rt[1] - t0) / 1e3:9.1f}")
    if os.environ.get("PH_DUMP"):
        np.savetxt(os.environ["PH_DUMP"], rel, fmt="%.1f")
    ctas = max(c[15], 1)
    print(json.dumps({"config": args.config, "plan": tp.last_plan(), "us_per_launch": s.elapsed_time(e) * 1e3 / args.reps,
                      "cycles_per_cta": {SLOTS[i]: round(c[i] / ctas) for i in range(16)}}, indent=1))


if __name__ == "__main__":
    main()
