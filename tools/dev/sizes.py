import sys, torch, numpy as np, os
sys.path.insert(0, os.getcwd())
import paper_2001_04438_b200 as tp, workloads
for logn in (26, 27, 28, 29, 31):
    n = 1 << logn
    x = torch.from_numpy(workloads.generate("c5", ncols=n)).cuda()
    ws = tp.new_workspace(*x.shape)
    y = torch.empty_like(x)
    p = tp.partial(x, workspace=ws).reshape(1, 1, 2).contiguous()
    res = []
    for nm, fn in [("full", lambda s: tp.softmax_ex(x, out=y, workspace=ws, schedule=s)),
                   ("partial", lambda s: tp.partial(x, workspace=ws, schedule=s)),
                   ("finish", lambda s: tp.finish(x, p, 1, out=y, workspace=ws, schedule=s))]:
        for s in (1, 5):
            for _ in range(3): fn(s)
            torch.cuda.synchronize()
            ts = []
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); fn(s); b.record(); ts.append((a, b))
            torch.cuda.synchronize()
            res.append(f"{nm}{'ST' if s == 1 else 'PH'}={np.median([a.elapsed_time(b) * 1e3 for a, b in ts]):.1f}")
    print(f"2^{logn}", " ".join(res), flush=True)
    del x, y, ws
    torch.cuda.empty_cache()
