import sys, json, torch, numpy as np, os, subprocess
ROOT = os.getcwd()
CHILD = r"""
import sys, torch, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2001_04438_b200 as tp, workloads
x = torch.from_numpy(workloads.generate(sys.argv[2])).cuda()
ws = tp.new_workspace(*x.shape)
y = torch.empty_like(x)
out = []
for what in sys.argv[3].split(","):
    sched = 5 if what.endswith("ph") else 1
    fn = (lambda: tp.partial(x, workspace=ws, schedule=sched)) if what.startswith("p1") else (lambda: tp.softmax_ex(x, out=y, workspace=ws, schedule=sched))
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    out.append(f"{what}={np.median([a.elapsed_time(b) * 1e3 for a, b in ts]):.1f}")
print(" ".join(out))
"""
libs = sys.argv[1].split(",")
cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
whats = sys.argv[3] if len(sys.argv) > 3 else "p1st,p1ph,fullst,fullph"
for rnd in range(int(sys.argv[4]) if len(sys.argv) > 4 else 3):
    for l in libs:
        env = dict(os.environ, TP_LIBRARY=os.path.abspath(l))
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, cfg, whats], env=env, capture_output=True, text=True)
        print(rnd, os.path.basename(l)[-28:], r.stdout.strip() or r.stderr[-300:], flush=True)
