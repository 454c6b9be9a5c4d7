import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2001_04438_b200 as tp, workloads
for lg in [int(v) for v in sys.argv[1].split(",")]:
    for cfg in sys.argv[2].split(","):
        x = torch.from_numpy(workloads.generate(cfg, ncols=1 << lg)).cuda()
        ws = tp.new_workspace(*x.shape)
        for it in range(3):
            tp.partial(x, workspace=ws, schedule=5)
            torch.cuda.synchronize()
        print(cfg, lg, "partial ok", flush=True)
        for it in range(3):
            y = tp.softmax_ex(x, schedule=5)
            torch.cuda.synchronize()
        print(cfg, lg, "full ok", flush=True)
        del x, y
