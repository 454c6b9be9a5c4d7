"""Alternating A/B timing of library builds (development tool).

    python tools/ab_libs.py --libs a.so,b.so --configs c5,c3 [--rounds 4] [--reps 10] [--schedule 0]

Each round runs every library once per config in a fresh subprocess (TP_LIBRARY), K back-to-back
launches timed with CUDA events; prints the per-library median of the round medians.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, torch, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2001_04438_b200 as tp, workloads
cfg, reps, sched, algo = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
x = workloads.generate(cfg)
xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
y = torch.empty(xd.shape, dtype=torch.float32, device="cuda")
ws = tp.new_workspace(*xd.shape)
for _ in range(3):
    tp.softmax_ex(xd, algo, out=y, workspace=ws, schedule=sched)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); tp.softmax_ex(xd, algo, out=y, workspace=ws, schedule=sched); b.record()
    ts.append((a, b))
torch.cuda.synchronize()
print(json.dumps({"us": float(np.median([a.elapsed_time(b) * 1e3 for a, b in ts])), "plan": tp.last_plan()}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--configs", default="c5,c3")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--schedule", type=int, default=0)
    ap.add_argument("--algo", type=int, default=0)
    args = ap.parse_args()
    libs = args.libs.split(",")
    res = {(l, c): [] for l in libs for c in args.configs.split(",")}
    for _ in range(args.rounds):
        for c in args.configs.split(","):
            for l in libs:
                env = dict(os.environ, TP_LIBRARY=os.path.abspath(l))
                r = subprocess.run([sys.executable, "-c", CHILD, ROOT, c, str(args.reps), str(args.schedule),
                                    str(args.algo)], env=env, capture_output=True, text=True, timeout=600)
                if r.returncode:
                    print(l, c, "FAILED", r.stderr[-500:])
                    continue
                d = json.loads(r.stdout.strip().splitlines()[-1])
                res[(l, c)].append(d["us"])
    for (l, c), v in res.items():
        v = sorted(v)
        print(f"{c:4s} {os.path.basename(l):45s} median {v[len(v) // 2]:9.1f} us  all {[round(t, 1) for t in v]}")


if __name__ == "__main__":
    main()
