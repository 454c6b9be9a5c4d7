"""Host-side cost of one launch through the binding and through the raw C ABI (development)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402

x = torch.randn(64, 32768, device="cuda")
y = torch.empty_like(x)
L = tp.lib()
st = torch.cuda.current_stream().cuda_stream


def bench(name, fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:40s} host {1e6 * (t1 - t0) / n:8.2f} us/call   incl. drain {1e6 * (t2 - t0) / n:8.2f} us/call")


bench("tp.softmax_ex(x, out=y)", lambda: tp.softmax_ex(x, out=y))
bench("tp.softmax(x)", lambda: tp.softmax(x))
bench("L.softmax_f32 raw ctypes", lambda: L.softmax_f32(x.data_ptr(), y.data_ptr(), 64, 32768, st))
bench("L.softmax_ex raw ctypes", lambda: L.softmax_ex(0, 0, x.data_ptr(), y.data_ptr(), 64, 32768, None, 0, None, st))
bench("L.softmax_ex stream sched", lambda: L.softmax_ex(0, 0, x.data_ptr(), y.data_ptr(), 64, 32768, None, 0,
                                                        tp._opts(schedule=1), st))
bench("torch.softmax (reference point)", lambda: torch.softmax(x, -1))
bench("ctypes no-op (softmax_status_str)", lambda: L.softmax_status_str(0))
