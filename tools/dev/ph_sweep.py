"""Phase kernel on many rows (interleaved order): time C4 / C4b for several lookaheads (development)."""
import hashlib
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2001_04438_b200 as tp, workloads

Ls = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 4, 8, 12, 16, 24, 32, 48]
for cfg in sys.argv[1].split(","):
    x = workloads.generate(cfg)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    ws = tp.new_workspace(*xd.shape)
    ref = tp.softmax_ex(xd, schedule=tp.SCHED_STREAM)
    href = hashlib.sha1(ref.view(torch.int32).cpu().numpy().tobytes()).hexdigest()[:12]
    for name, kw in [("auto", {})] + [(f"ph L={L}", dict(schedule=tp.SCHED_PHASE, lookahead_rows=L)) for L in Ls]:
        for _ in range(3):
            tp.softmax_ex(xd, out=y, workspace=ws, **kw)
        torch.cuda.synchronize()
        h = hashlib.sha1(y.view(torch.int32).cpu().numpy().tobytes()).hexdigest()[:12]
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); tp.softmax_ex(xd, out=y, workspace=ws, **kw); b.record(); ts.append((a, b))
        torch.cuda.synchronize()
        print(cfg, name, round(float(np.median([a.elapsed_time(b) * 1e3 for a, b in ts])), 1), "same" if h == href else "DIFF",
              tp.last_plan(), tp.watchdog_flags(), flush=True)
