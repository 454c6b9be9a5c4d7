"""Step-by-step diagnostic run (prints and flushes after every step; development tool).

    python tools/diag.py c2:recompute c3:two_pass ...
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.time()


def say(*a):
    print(f"[{time.time() - t0:7.2f}s]", *a, flush=True)


import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

ALGO = {"two_pass": tp.ALGO_TWO_PASS, "recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}
torch.zeros(1, device="cuda")
tp.lib()
say("ready")
for spec in sys.argv[1:] or ["c1:two_pass", "c2:two_pass", "c2:recompute", "c2:reload"]:
    key, algo = spec.split(":")[:2]
    opts = dict(kv.split("=") for kv in spec.split(":")[2:])
    opts = {k: int(v) for k, v in opts.items()}
    x = workloads.generate(key)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else \
        torch.from_numpy(x).cuda()
    say(spec, x.shape, "launch")
    y = tp.softmax_ex(xd, ALGO[algo], **opts)
    torch.cuda.synchronize()
    say(spec, "done; watchdog", tp.watchdog_flags())
    if x.size <= 50_000_000:
        say(spec, "check", oracle.check_rows(x, y.cpu().numpy()))
