"""PCIe bounds for the end-to-end (host buffer) path: pinned H2D, D2H, and both at once."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa

n = 256 * 800000
hx = torch.empty(n, dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
dx = torch.empty(n, dtype=torch.float32, device="cuda")
dy = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, k=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3


h2d = t(lambda: dx.copy_(hx, non_blocking=True))
d2h = t(lambda: hy.copy_(dy, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)


bo = t(both)
e2e = t(lambda: tp.softmax_host(hx.view(256, 800000), hy.view(256, 800000)))
gb = n * 4 / 1e9
print(f"H2D {h2d:.2f} ms ({gb / h2d * 1e3:.1f} GB/s)  D2H {d2h:.2f} ms ({gb / d2h * 1e3:.1f} GB/s)  "
      f"both {bo:.2f} ms  softmax_host {e2e:.2f} ms")
