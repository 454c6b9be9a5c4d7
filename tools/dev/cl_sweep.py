"""Time C4 / C4b on forced schedules and cluster sizes (development)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2001_04438_b200 as tp, workloads

for cfg in sys.argv[1].split(","):
    x = workloads.generate(cfg)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    ws = tp.new_workspace(*xd.shape)
    for name, kw in [("auto", {}), ("stream", dict(schedule=tp.SCHED_STREAM)), ("cl1", dict(schedule=tp.SCHED_CLUSTER, cluster_size=1)),
                     ("cl2", dict(schedule=tp.SCHED_CLUSTER, cluster_size=2)), ("cl4", dict(schedule=tp.SCHED_CLUSTER, cluster_size=4)),
                     ("cl8", dict(schedule=tp.SCHED_CLUSTER, cluster_size=8)), ("cl16", dict(schedule=tp.SCHED_CLUSTER, cluster_size=16))]:
        try:
            for _ in range(3):
                tp.softmax_ex(xd, out=y, workspace=ws, **kw)
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); tp.softmax_ex(xd, out=y, workspace=ws, **kw); b.record(); ts.append((a, b))
            torch.cuda.synchronize()
            print(cfg, name, round(float(np.median([a.elapsed_time(b) * 1e3 for a, b in ts])), 1), tp.last_plan(), flush=True)
        except Exception as e:
            print(cfg, name, "ERR", str(e)[:100])
