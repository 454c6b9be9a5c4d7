"""Step-by-step diagnostic run (prints and flushes after every step)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.time()
def say(*a):
    print(f"[{time.time()-t0:7.2f}s]", *a, flush=True)
import torch
say("torch", torch.__version__, torch.cuda.is_available())
torch.zeros(1, device="cuda"); torch.cuda.synchronize(); say("cuda init")
import paper_2001_04438_b200 as tp, workloads, oracle
tp.lib(); say("lib loaded")
import numpy as np
for key, rows, cols, kw in [("c1", None, None, {}), ("c1", None, None, dict(force_persistent=True)),
                            ("c2", 4, None, {}), ("c2", None, None, {}), ("c3", None, None, {})]:
    x = workloads.generate(key, nrows=rows, ncols=cols)
    xd = torch.from_numpy(x).cuda()
    say(key, x.shape, kw, "launch")
    y = tp.softmax_ex(xd, **kw)
    torch.cuda.synchronize()
    say(key, "done; watchdog", tp.watchdog_flags())
    r = oracle.check_rows(x, y.cpu().numpy())
    say(key, "check", r)
