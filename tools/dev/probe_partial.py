import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2001_04438_b200 as tp, workloads
for n in [16384 * 200, 16384 * 148 * 48, 1 << 28, 1 << 31]:
    x = torch.from_numpy(workloads.generate("c5", ncols=n)).cuda()
    ws = tp.new_workspace(*x.shape)
    y = torch.empty_like(x)
    for nm, fn in [("partial-ws", lambda: tp.partial(x, workspace=ws, schedule=5)),
                   ("full", lambda: tp.softmax_ex(x, out=y, schedule=5)),
                   ("full-ws", lambda: tp.softmax_ex(x, out=y, workspace=ws, schedule=5))]:
        try:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            print(n, nm, "ok", tp.last_plan()["kernel"], flush=True)
        except Exception as e:
            print(n, nm, "FAIL", e, flush=True)
            sys.exit(1)
