"""Print a hash of the softmax output of a config under the library in TP_LIBRARY (development)."""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

for cfg in sys.argv[1].split(","):
    sched = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    x = workloads.generate(cfg)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
    y = tp.softmax_ex(xd, schedule=sched)
    torch.cuda.synchronize()
    h = hashlib.sha1(y.view(torch.int32).cpu().numpy().tobytes()).hexdigest()[:16]
    print(cfg, sched, h, tp.last_plan(), tp.watchdog_flags())
