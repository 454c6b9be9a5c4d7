"""C1 / C2 timing of the small schedule by cluster size (development tool).

    python tools/small_ab.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

for key in ("c2", "c1"):
    x = torch.from_numpy(workloads.generate(key)).cuda()
    y = torch.empty_like(x)
    ws = tp.new_workspace(*x.shape)
    for cl in (0, 1, 2, 3):
        fn = lambda: tp.softmax_ex(x, out=y, workspace=ws, schedule=tp.SCHED_SMALL, cluster_size=cl)  # noqa
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        # back to back, and device time per call from a CUDA graph of 20 calls
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            fn()
        b.record()
        b.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    fn()
        g.replay()
        torch.cuda.synchronize()
        c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c.record()
        g.replay()
        d.record()
        d.synchronize()
        print(json.dumps({"cfg": key, "cluster_size": cl, "plan": tp.last_plan(), "b2b_us": round(a.elapsed_time(b) * 1e3 / 50, 2),
                          "graph_us": round(c.elapsed_time(d) * 1e3 / 20, 2)}), flush=True)
