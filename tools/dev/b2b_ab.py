"""Back-to-back (bench-style) A/B of launch options on one workload (development tool).

    python tools/b2b_ab.py c4 'schedule=1' 'schedule=3,cluster_size=4' 'schedule=3,cluster_size=8'
"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa
import workloads  # noqa

key = sys.argv[1]
cands = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in c.split(",") if kv) for c in sys.argv[2:]]
x = workloads.generate(key)
xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
ws = tp.new_workspace(*xd.shape)
res = {i: [] for i in range(len(cands))}
for rnd in range(6):
    for i, c in enumerate(cands):
        for _ in range(3):
            tp.softmax_ex(xd, out=y, workspace=ws, **c)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            tp.softmax_ex(xd, out=y, workspace=ws, **c)
        b.record()
        b.synchronize()
        res[i].append(a.elapsed_time(b) * 1e3 / 20)
assert tp.watchdog_flags(ws) == 0
for i, c in enumerate(cands):
    v = np.array(res[i])
    print(json.dumps({"cfg": key, "opts": c, "median_us": round(float(np.median(v)), 1), "min_us": round(float(v.min()), 1),
                      "max_us": round(float(v.max()), 1)}))
