"""Repeat the host-pipeline slab test's call sequence and report where a result differs (development tool)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2001_04438_b200 as tp, workloads
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
xb = workloads.generate("c4b", 0, 200)
hxb = torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).pin_memory()
xf = workloads.generate("c4", 0, 100)
hxf = torch.from_numpy(xf).pin_memory()
refb = tp.softmax(hxb.cuda()).cpu().numpy()
reff = tp.softmax(torch.from_numpy(xf).cuda()).cpu().numpy()
bad = 0
for it in range(iters):
    for name, hx, ref in (("bf16", hxb, refb), ("fp32", hxf, reff)):
        hy = tp.softmax_host(hx).numpy()
        if not np.array_equal(hy, ref):
            bad += 1
            r, c = np.nonzero(hy != ref)
            rows = np.unique(r)
            print(it, name, "host differs: rows", rows[:20], "n", len(r), "cols", c.min(), c.max(), flush=True)
        dev = tp.softmax(hx.cuda()).cpu().numpy()
        if not np.array_equal(dev, ref):
            bad += 1
            r, c = np.nonzero(dev != ref)
            print(it, name, "device differs: rows", np.unique(r)[:20], "n", len(r), "cols", c.min(), c.max(), flush=True)
print("iters", iters, "bad", bad, "watchdog", tp.watchdog_flags() if hasattr(tp, "watchdog_flags") else None)
