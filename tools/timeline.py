"""Per-CTA timeline of the stream kernel (development tool): start, first later-phase item
taken, its row statistics first seen, queue exhaustion, exit.

    python tools/timeline.py c3 [partial|two_pass]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

key = sys.argv[1]
what = sys.argv[2] if len(sys.argv) > 2 else "two_pass"
x = torch.from_numpy(workloads.generate(key)).cuda()
y = torch.empty_like(x)
ws = tp.new_workspace(*x.shape)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
run = (lambda: tp.partial(x, workspace=ws)) if what == "partial" else \
    (lambda: tp.softmax_ex(x, out=y, workspace=ws, schedule=tp.SCHED_STREAM))
for _ in range(3):
    run()
buf = torch.zeros(16 + 5 * 1024, dtype=torch.int64, device="cuda")
flush.zero_()
tp.lib().tp_set_profile_buffer(buf.data_ptr())
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
mark = torch.zeros(4, dtype=torch.float32, device="cuda")
m2 = torch.zeros(4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
s.record()
tp.lib().tp_debug_op(5, mark.data_ptr(), None, mark.data_ptr(), None, 1, st)   # marker before
run()
tp.lib().tp_debug_op(5, m2.data_ptr(), None, m2.data_ptr(), None, 1, st)       # marker after
e.record()
e.synchronize()
tp.lib().tp_set_profile_buffer(None)
b = buf.cpu().numpy()[16:].reshape(-1, 5)
b = b[b[:, 0] > 0].astype(np.float64)
t0 = float(mark.cpu().numpy().view(np.int64)[0])
t_after = (float(m2.cpu().numpy().view(np.int64)[0]) - t0) / 1e3
st, ex, en = (b[:, 0] - t0) / 1e3, (b[:, 1] - t0) / 1e3, (b[:, 2] - t0) / 1e3
p2, rel = (b[:, 3] - t0) / 1e3, (b[:, 4] - t0) / 1e3


def q(v):
    v = v[v > -1e6]
    return [round(float(np.min(v)), 2), round(float(np.median(v)), 2), round(float(np.max(v)), 2)] if len(v) else None
print(json.dumps({"config": key, "what": what, "event_us": s.elapsed_time(e) * 1e3, "ctas": len(b),
                  "marker_after_us": round(t_after, 2),
                  "start_us": [round(float(np.min(st)), 2), round(float(np.median(st)), 2), round(float(np.max(st)), 2)],
                  "p2_taken_us": q(p2), "released_seen_us": q(rel),
                  "exhausted_us": [round(float(np.min(ex)), 2), round(float(np.median(ex)), 2), round(float(np.max(ex)), 2)],
                  "exit_us": [round(float(np.min(en)), 2), round(float(np.median(en)), 2), round(float(np.max(en)), 2)]}))
