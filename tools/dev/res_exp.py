"""Time (library, lookahead) combinations of the resident-row kernel on one config (development tool).

    python tools/dev/res_exp.py c4b exp_libs/exp0.so:0 exp_libs/exp14.so:2[:schedule[:cluster_size]] ...
"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r"""
import sys, json, torch, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2001_04438_b200 as tp, workloads
cfg, la, sched, cs = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
x = workloads.generate(cfg)
xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
ws = tp.new_workspace(*xd.shape)
for _ in range(3):
    tp.softmax_ex(xd, 0, out=y, workspace=ws, lookahead_rows=la, schedule=sched, cluster_size=cs)
torch.cuda.synchronize()
ts = []
for _ in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); tp.softmax_ex(xd, 0, out=y, workspace=ws, lookahead_rows=la, schedule=sched, cluster_size=cs); b.record()
    ts.append((a, b))
torch.cuda.synchronize()
print(json.dumps({"us": float(np.median([a.elapsed_time(b) * 1e3 for a, b in ts])), "plan": tp.last_plan()}))
"""
cfg = sys.argv[1]
for spec in sys.argv[2:]:
    lib, la, sched, cs = (spec.split(":") + ["0", "0"])[:4]
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, cfg, la, sched, cs], env=dict(os.environ, TP_LIBRARY=os.path.abspath(lib)),
                       capture_output=True, text=True, timeout=600)
    if r.returncode:
        print(spec, "FAILED", r.stderr[-400:]); continue
    d = json.loads(r.stdout.strip().splitlines()[-1])
    print(f"{spec:32s} {d['us']:8.1f} us  plan {d['plan']}", flush=True)
