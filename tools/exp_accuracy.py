"""Exhaustive ULP metrology of the device exponentials ("maximum
error under 2 ULP, validated through exhaustive evaluation on all valid inputs").

    python tools/exp_accuracy.py [--json out.json] [--stride 1]

Every fp32 input of each domain (stride 1 = exhaustive) goes through tp_exp_sweep on the GPU;
the reference is float64 on the host (error < 1e-9 ulp of fp32, far below what is measured):
  exp      Alg. 4 (Three-Pass Exp) on x in [ln FLT_MIN, 0] (normal outputs, the comparators'
           domain x - mu <= 0, PAPER.md:258 footnote): ulp error of y against e^x;
  extexp   ExtExp on |x| <= 2^21 (reading G11): ulp error of m against e^(x - n ln 2), n the
           exponent the GPU returned (the pair must represent e^x = m 2^n).
Measurement only: the parity tests grade outputs against the oracle (tests/).
"""
import argparse
import json
import math
import os
import struct
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402

CHUNK = 1 << 24


def f2b(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def ulp32(v):
    """ulp of the fp32 value nearest v (v > 0, normal), float64 array."""
    e = np.floor(np.log2(v))
    return np.exp2(e - 23)


def sweep(what, lo_bits, hi_bits, stride, stream):
    """Inclusive bit range [lo_bits, hi_bits]; returns stats."""
    L = tp.lib()
    o0 = torch.empty(CHUNK, dtype=torch.float32, device="cuda")
    o1 = torch.empty(CHUNK, dtype=torch.float32, device="cuda")
    hist = np.zeros(8, np.int64)  # ulp bins: <=0.5, <=1, <=1.5, <=2, <=2.5, <=3, <=4, >4
    edges = np.array([0.5, 1.0, 1.5, 2.0, 2.5, 3.0, 4.0])
    worst, worst_x, n_total, sum_err = 0.0, None, 0, 0.0
    b = lo_bits
    while b <= hi_bits:
        cnt = min(CHUNK * stride, hi_bits - b + 1)
        assert L.tp_exp_sweep(what, b, cnt, o0.data_ptr(), o1.data_ptr(), stream) == 0
        torch.cuda.synchronize()
        m = o0[:cnt].cpu().numpy()[::stride].astype(np.float64)
        bits = (np.arange(0, cnt, stride, dtype=np.uint64) + np.uint64(b)).astype(np.uint32)
        x = bits.view(np.float32).astype(np.float64)
        if what == 0:
            n = o1[:cnt].cpu().numpy()[::stride].astype(np.float64)
            ref = np.exp(x - n * math.log(2.0))
        else:
            ref = np.exp(x)
        err = np.abs(m - ref) / ulp32(ref)
        i = int(np.argmax(err))
        if err[i] > worst:
            worst, worst_x = float(err[i]), float(x[i])
        hist += np.bincount(np.searchsorted(edges, err), minlength=8)[:8]
        n_total += err.size
        sum_err += float(err.sum())
        b += cnt
    return {"inputs": n_total, "max_ulp": worst, "worst_x": worst_x, "mean_ulp": sum_err / max(n_total, 1),
            "hist_ulp_le": dict(zip(["0.5", "1", "1.5", "2", "2.5", "3", "4", ">4"], hist.tolist()))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--stride", type=int, default=1)
    args = ap.parse_args()
    stream = torch.cuda.current_stream().cuda_stream
    res = {"stride": args.stride}
    t0 = time.time()
    lnmin = math.log(np.finfo(np.float32).tiny)  # -87.3365...
    lo = np.float32(lnmin)
    if float(lo) < lnmin:
        lo = np.nextafter(lo, np.float32(0))
    # negative floats: bits grow with |x|: [-0 .. lo]
    res["exp"] = sweep(1, f2b(-0.0), f2b(float(lo)), args.stride, stream)
    res["exp"]["domain"] = f"[{float(lo)}, 0]"
    print(json.dumps({"exp": res["exp"]}), flush=True)
    # ExtExp by |x| band: the configurations' domain (|x| <= 1e4) and the clamp domain (2^21)
    prev = 0.0
    for name, lim in (("extexp_abs_le_1e4", 1e4), ("extexp_1e4_to_2p21", float(2 ** 21))):
        lo_b = f2b(prev) if prev == 0.0 else f2b(float(np.nextafter(np.float32(prev), np.float32(np.inf))))
        a = sweep(0, lo_b, f2b(lim), args.stride, stream)
        lo_n = f2b(-0.0) if prev == 0.0 else f2b(-float(np.nextafter(np.float32(prev), np.float32(np.inf))))
        bneg = sweep(0, lo_n, f2b(-lim), args.stride, stream)
        hist = {k: a["hist_ulp_le"][k] + bneg["hist_ulp_le"][k] for k in a["hist_ulp_le"]}
        worst = a if a["max_ulp"] >= bneg["max_ulp"] else bneg
        res[name] = {"inputs": a["inputs"] + bneg["inputs"], "max_ulp": worst["max_ulp"], "worst_x": worst["worst_x"],
                     "mean_ulp": (a["mean_ulp"] * a["inputs"] + bneg["mean_ulp"] * bneg["inputs"]) /
                     (a["inputs"] + bneg["inputs"]), "hist_ulp_le": hist,
                     "domain": f"{prev} < |x| <= {lim}" if prev else f"|x| <= {lim}"}
        print(json.dumps({name: res[name]}), flush=True)
        prev = lim
    res["seconds"] = time.time() - t0
    if args.json:
        json.dump(res, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
