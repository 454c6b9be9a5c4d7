"""HBM read throughput by access method (development / roofline evidence).

    python tools/read_probe.py [out.json]

Reads a 1 GiB buffer (out of L2) with: LDG.128 grid-stride at 4 / 8 / 16 loads in flight per
thread, and bulk (TMA) copies into shared memory with several chunk sizes x ring depths x CTAs
per SM.  Prints GB/s (median of 10 timed launches, CUDA events, back to back).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def main():
    L = tp.lib()
    nbytes = 1 << 30
    x = torch.ones(nbytes // 4, dtype=torch.float32, device="cuda")
    sink = torch.zeros(148 * 8, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = []
    for what, name in ((3, "ldg128_x4"), (4, "ldg128_x8"), (5, "ldg128_x16")):
        for cps in (2, 4):
            t = timed(lambda: L.tp_stream_baseline(what, x.data_ptr(), sink.data_ptr(), x.numel(), 1.0, cps * sms, st))
            out.append({"method": name, "ctas": cps * sms, "GBps": round(nbytes / t / 1e9, 1)})
            print(json.dumps(out[-1]), flush=True)
    for chunk_kb, stages, cps in ((64, 3, 1), (32, 6, 1), (16, 12, 1), (8, 24, 1), (16, 6, 2), (32, 3, 2),
                                  (64, 2, 1), (32, 4, 1), (16, 8, 1), (48, 4, 1), (4, 32, 1), (8, 12, 2),
                                  (16, 4, 3), (16, 3, 4)):
        ctas = cps * sms
        t = timed(lambda: L.tp_read_probe(x.data_ptr(), nbytes, chunk_kb << 10, stages, ctas, sink.data_ptr(), st))
        rc = L.tp_read_probe(x.data_ptr(), nbytes, chunk_kb << 10, stages, ctas, sink.data_ptr(), st)
        assert rc == 0, rc
        out.append({"method": "tma_bulk", "chunk_kb": chunk_kb, "stages": stages, "ctas_per_sm": cps,
                    "inflight_kb_per_sm": chunk_kb * stages * cps, "GBps": round(nbytes / t / 1e9, 1)})
        print(json.dumps(out[-1]), flush=True)
    torch.cuda.synchronize()
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
