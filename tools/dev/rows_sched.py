import sys, json, torch, numpy as np
sys.path.insert(0, '.')
import paper_2001_04438_b200 as tp, workloads
def timed(fn, reps=15):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ev=[]
    for _ in range(reps):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); a.record(); fn(); b.record(); ev.append((a,b))
    torch.cuda.synchronize(); return float(np.median([a.elapsed_time(b)*1e3 for a,b in ev]))
for key in ['c4','c4b']:
  for r in [32, 64]:
    x = workloads.generate(key, row0=0, nrows=r)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
    y = torch.empty(xd.shape, dtype=torch.float32, device='cuda')
    out = {}
    for name, sched, cl in [('auto',0,0),('stream',1,0),('phase',5,0),('cl2',3,2),('cl4',3,4),('cl8',3,8),('cl16',3,16)]:
        try:
            t = timed(lambda: tp.softmax_ex(xd, out=y, schedule=sched, cluster_size=cl))
            out[name] = (round(t,1), tp.last_plan()['kernel'], tp.last_plan()['grid_ctas'])
        except Exception as e:
            out[name] = str(e)[:40]
    print(key, r, json.dumps(out), flush=True)
