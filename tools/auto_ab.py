"""Back-to-back timing of the AUTO schedule on given configs with whichever library TP_LIBRARY
names (development tool; pair with a TP_DEV_OVERRIDES build and its environment switches)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402
from tools.res_ab import BYTES, timed  # noqa: E402

for key in (sys.argv[1] if len(sys.argv) > 1 else "c4b,c4").split(","):
    cfg = workloads.CONFIGS[key]
    x = workloads.generate(key)
    xd = (torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if cfg.dtype == "bf16"
          else torch.from_numpy(x).cuda())
    y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
    ws = tp.new_workspace(*xd.shape)
    tp.softmax_ex(xd, out=y, workspace=ws)
    plan = tp.last_plan()
    us = min(timed(lambda: tp.softmax_ex(xd, out=y, workspace=ws), 20) for _ in range(3))
    print(json.dumps(dict(config=key, lib=os.environ.get("TP_LIBRARY", "release"), env_resident=os.environ.get("TP_RESIDENT"),
                          plan=plan, us=us, alg_GBps=BYTES[cfg.dtype] * cfg.elements / (us * 1e-6) / 1e9,
                          watchdog=tp.watchdog_flags(ws))), flush=True)
