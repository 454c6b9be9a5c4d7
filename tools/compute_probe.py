"""Compute-only time per block of the per-block operations (development / roofline evidence).

    python tools/compute_probe.py [--ctas 148] [--reps 200]

Runs tp_bench_compute (libtwopass.so) for pass 1, pass 2 and both, fp32 and bf16, and prints
microseconds per 16384-element block per SM: the floor the block operations put under any
schedule (HBM budget at 6.45 TB/s over 148 SMs: 8 B/elem -> 3.0 us, 12 B/elem -> 4.5 us).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04438_b200 as tp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctas", type=int, default=148)
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    sink = torch.empty(args.ctas * 16 + args.ctas * 16384, dtype=torch.float32, device="cuda")
    L = tp.lib()
    st = torch.cuda.current_stream().cuda_stream
    for dt, name in ((0, "f32"), (1, "bf16")):
        ops = ((0, "pass1"), (1, "pass2"), (2, "both"))
        if dt == 0:
            ops += ((3, "ffma2"), (4, "ffma2_imm"), (5, "ffma"), (6, "alu_addmax_shf"), (7, "pass1_thread"), (8, "pass2_with_stores"),
                    (9, "stores_only"),
                    (10, "stores_via_smem_tma"), (11, "stores_256bit"))
        for what, wn in ops:
            for _ in range(2):
                assert L.tp_bench_compute(what, dt, args.ctas, args.reps, sink.data_ptr(), st) == 0
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            assert L.tp_bench_compute(what, dt, args.ctas, args.reps, sink.data_ptr(), st) == 0
            e.record()
            e.synchronize()
            us = s.elapsed_time(e) * 1e3
            extra = {}
            if 3 <= what <= 6:  # warp-instructions per clock per SM (64 per thread per rep, 16 warps per CTA)
                extra["warp_inst_per_clk_per_sm_at_1965MHz"] = 64 * 16 * args.reps / (us * 1e-6) / 1.965e9
            print(json.dumps({"in": name, "op": wn, "ctas": args.ctas, "reps": args.reps, **extra,
                              "us_per_block_per_sm": us / args.reps,
                              "elems_per_s": args.ctas * args.reps * 16384 / (us * 1e-6)}), flush=True)


if __name__ == "__main__":
    main()
