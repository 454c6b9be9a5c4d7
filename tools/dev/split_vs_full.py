"""C5: the Two-Pass as one phase-kernel launch vs partial (phase) + finish (stream / phase) (development)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2001_04438_b200 as tp, workloads

x = torch.from_numpy(workloads.generate(sys.argv[1] if len(sys.argv) > 1 else "c5")).cuda()
y = torch.empty_like(x)
ws = tp.new_workspace(*x.shape)
pairs = torch.empty((1, x.shape[0], 2), dtype=torch.float32, device="cuda")
fns = {
    "full_phase": lambda: tp.softmax_ex(x, out=y, workspace=ws, schedule=tp.SCHED_PHASE),
    "partial_ph+finish_st": lambda: (tp.partial(x, out=pairs[0], workspace=ws, schedule=tp.SCHED_PHASE),
                                     tp.finish(x, pairs, 1, out=y, workspace=ws, schedule=tp.SCHED_STREAM)),
    "partial_ph+finish_ph": lambda: (tp.partial(x, out=pairs[0], workspace=ws, schedule=tp.SCHED_PHASE),
                                     tp.finish(x, pairs, 1, out=y, workspace=ws, schedule=tp.SCHED_PHASE)),
    "finish_st": lambda: tp.finish(x, pairs, 1, out=y, workspace=ws, schedule=tp.SCHED_STREAM),
    "finish_ph": lambda: tp.finish(x, pairs, 1, out=y, workspace=ws, schedule=tp.SCHED_PHASE),
}
for rnd in range(3):
    out = []
    for k, fn in fns.items():
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); ts.append((a, b))
        torch.cuda.synchronize()
        out.append(f"{k}={np.median([a.elapsed_time(b) * 1e3 for a, b in ts]):.1f}")
    print(rnd, " ".join(out), flush=True)
