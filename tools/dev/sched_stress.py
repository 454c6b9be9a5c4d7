"""Repeat AUTO / STREAM / CLUSTER calls on C4-like fp32 shapes with one workspace and report where results
differ from the first STREAM result (development tool: hunting a rare mismatch seen in the GPU suite)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2001_04438_b200 as tp, workloads
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rows, cols = 256, 16384 * 49 + 5000
x = workloads.ragged_case(rows, cols, -400, 400, seed=18, stream=rows)
xd = torch.from_numpy(x).cuda()
ws = tp.new_workspace(rows, cols)
refd = tp.softmax_ex(xd, workspace=ws, schedule=tp.SCHED_STREAM).clone()
ref = refd.cpu().numpy()
names = {tp.SCHED_AUTO: "auto", tp.SCHED_STREAM: "stream", tp.SCHED_CLUSTER: "cluster"}
bad = 0
for it in range(iters):
    for sched in (tp.SCHED_AUTO, tp.SCHED_STREAM, tp.SCHED_CLUSTER):
        yd = tp.softmax_ex(xd, workspace=ws, schedule=sched)
        plan = tp.last_plan()
        if torch.equal(yd.view(torch.int32), refd.view(torch.int32)):
            continue
        y = yd.cpu().numpy()
        if True:
            bad += 1
            r, c = np.nonzero(y != ref)
            rel = np.abs(y[r, c].astype(np.float64) - ref[r, c]) / np.maximum(np.abs(ref[r, c]), 1e-300)
            print(it, names[sched], plan, "rows", np.unique(r)[:12].tolist(), "n", len(r), "cols", int(c.min()), int(c.max()),
                  "blocks", np.unique(c // 16384)[:12].tolist(), "max rel", float(rel.max()), "wd", tp.watchdog_flags(ws), flush=True)
print("iters", iters, "bad", bad)
