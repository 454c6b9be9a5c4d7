"""HBM copy ceiling on B200 (measurement): y = x with bulk (TMA) copies both ways (tp_copy_probe),
against torch's copy_ and pass 2 of the Two-Pass on the same bytes (read x, write y).

    python tools/copy_probe.py [--gib 8]

Prints GB/s counting read + write bytes, median of 5 after a warm-up.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ts])) * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=8.0)
    args = ap.parse_args()
    n = int(args.gib * (1 << 30)) // 4
    x = torch.rand(n, device="cuda")
    y = torch.empty_like(x)
    nbytes = 2 * 4 * n
    s = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = {"bytes_moved": nbytes}
    res["torch_copy"] = nbytes / timed(lambda: y.copy_(x)) / 1e9
    for chunk, stages, per_sm, back in [(65536, 3, 1, 0), (32768, 6, 1, 0), (16384, 12, 1, 0), (32768, 3, 2, 0),
                                        (65536, 3, 1, 1), (32768, 6, 1, 1), (16384, 6, 2, 0)]:
        fn = lambda: tp.lib().tp_copy_probe(x.data_ptr(), y.data_ptr(), 4 * n, chunk, stages, sms * per_sm, back,
                                            ctypes.c_void_p(s))
        res[f"tma_copy c{chunk // 1024}k s{stages} x{per_sm}{' back' if back else ''}"] = nbytes / timed(fn) / 1e9
    # pass 2 of the Two-Pass alone on the same x (finish with one rank's pair; stream schedule)
    pairs = torch.empty((1, 1, 2), dtype=torch.float32, device="cuda")
    xr = x.view(1, -1)
    tp.partial(xr, out=pairs[0])
    res["two_pass_pass2 (finish)"] = nbytes / timed(lambda: tp.finish(xr, pairs, 1, out=y.view(1, -1))) / 1e9
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}, indent=1))


if __name__ == "__main__":
    main()
