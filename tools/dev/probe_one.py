"""Run one tp_bench_compute case (for ncu): python tools/probe_one.py WHAT [ctas] [reps] [bf16]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402

what = int(sys.argv[1])
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 148
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
dt = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sink = torch.empty(ctas * 16 + ctas * 16384, dtype=torch.float32, device="cuda")
for _ in range(2):
    assert tp.lib().tp_bench_compute(what, dt, ctas, reps, sink.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
print("ok")
