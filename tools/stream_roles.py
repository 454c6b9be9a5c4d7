"""Cycle accounting of the stream kernel's compute warp 0 (development tool).

    python tools/stream_roles.py c3 [two_pass|partial|phase<algo>_<phase>]

Installs a counter buffer (tp_set_profile_buffer), runs the stream schedule once after warm-up
and prints, per CTA and per block, where compute warp 0 spends its clock cycles: waiting for a
command, for the block's bulk copy, for a part slot, and in the pass-1 / later-phase work.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402
import workloads  # noqa: E402

SLOTS = ["cmd_wait", "data_wait", "part_wait", "p1_ops", "p2_ops", "total", "p1_blocks", "p2_blocks"]

key = sys.argv[1]
what = sys.argv[2] if len(sys.argv) > 2 else "two_pass"
x = torch.from_numpy(workloads.generate(key)).cuda()
y = torch.empty_like(x)
ws = tp.new_workspace(*x.shape)
if what.startswith("phase"):  # phase<algo>_<p>: one pass alone (tp_phase_only), e.g. phase2_0 = max pass
    algo, ph = (int(v) for v in what[5:].split("_"))
    tp.softmax_ex(x, algo, out=y, workspace=ws, schedule=tp.SCHED_STREAM)
    run = lambda: tp.phase_only(x, algo, ph, ws, out=y)  # noqa: E731
elif what == "partial":
    run = lambda: tp.partial(x, workspace=ws)  # noqa: E731
else:
    run = lambda: tp.softmax_ex(x, out=y, workspace=ws, schedule=tp.SCHED_STREAM)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
buf = torch.zeros(16 + 5 * 1024, dtype=torch.int64, device="cuda")
tp.lib().tp_set_profile_buffer(buf.data_ptr())
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
run()
e.record()
e.synchronize()
tp.lib().tp_set_profile_buffer(None)
bb = buf.cpu().tolist()
b = bb[:8]
prod = dict(zip(["chunk_switch", "issue", "cmd_slot_wait", "idle_passes", "total", "issued", "proxy_fence",
                "copy_issue"], bb[8:16]))
ctas = sum(1 for v in buf.cpu().numpy()[16:].reshape(-1, 5)[:, 0] if v > 0) or 1
blocks = max(b[6] + b[7], 1)
out = {"config": key, "what": what, "event_us": round(s.elapsed_time(e) * 1e3, 1), "ctas": ctas,
       "per_cta_kcycles": {k: round(v / ctas / 1e3, 1) for k, v in zip(SLOTS[:6], b[:6])},
       "per_block_cycles": {k: round(v / blocks) for k, v in zip(SLOTS[:6], b[:6])},
       "p1_ops_per_p1_block": round(b[3] / max(b[6], 1)), "p2_ops_per_p2_block": round(b[4] / max(b[7], 1)),
       "blocks": {"p1": b[6], "p2": b[7]},
       "producer_per_item_cycles": {k: round(v / max(prod["issued"], 1)) for k, v in prod.items() if k != "issued"}}
print(json.dumps(out))
