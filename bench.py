"""Benchmark of the Two-Pass softmax hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl ours|reference]

One step = one pass of the whole hot path (Alg. 3 pass 1 + pass 2) over one
batch of the workload, inputs resident in HBM.  Metric = BASELINE.json's: achieved HBM GB/s
under the paper's cost model (2 reads + 1 write = 12 B per fp32 element, Table 2
l.180-198), whole job, beside the in-house Three-Pass comparators on the same data.

Default workload: config 5 (one fp32 row of 2^31 elements, BASELINE.json configs[4]), the
largest single-GPU configuration and the one north_star defines multi-GPU throughput on:
  N = 1   the whole row on one GPU (one launch per step);
  N > 1   contiguous block-aligned chunks per rank (strong scaling): pass 1 per chunk, the
          ranks' 8-byte (m, n) partials all-gathered over NCCL (or --exchange nvlink /
          nvlink-fused: one-sided mailboxes), pass 2 per chunk; the Three-Pass comparators
          sharded the same way with their two all-gathers.
Beside it, every run also measures config 4 (256 x 800,000 fp32, and its bf16-input variant)
rows-sharded: 256/N rows per rank, no collective (`rows_sharded` in the JSON line).
Inputs are 8.6 GB (C5) / 819 MB (C4) per GPU at N = 1 > 126 MB L2: no explicit flush needed.

N > 1: launched by torchrun (one rank per GPU, NCCL).  Timing: W warm-up steps, then a barrier
+ synchronize, K steps between CUDA events on the launching stream, synchronize + barrier, max
over ranks.  Rank 0 prints one JSON line.

--impl reference: the reference arm for this tier is the oracle (oracle/, plain C, fp64 / long
double) on the host cores, rank 0 only, each step a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "two-pass softmax HBM GB/s and % of peak, vs three-pass, at 1/2/4/8 B200"
BYTES_PER_ELEM = {("two_pass", "f32"): 12, ("recompute", "f32"): 16, ("reload", "f32"): 20,
                  ("two_pass", "bf16"): 8, ("recompute", "bf16"): 10, ("reload", "bf16"): 16}
NOMINAL_HBM_GBS = 8000.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- clocks sampler

class ClockSampler:
    """nvidia-smi clocks + throttle reasons every 100 ms while running (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- workloads

def workload_spec(key: str, world: int, rank: int, scaling: str):
    """(description, rows, cols, dtype, generator(out_array) for this rank, elements this rank)."""
    import workloads
    from paper_2001_04438_b200 import dist as tpd
    cfg = workloads.CONFIGS[key]
    if cfg.rows == 1:
        # single long row: contiguous block-aligned chunks, one (m, n) all_gather (strong scaling)
        c0, c1 = tpd.chunk_range(cfg.cols, world, rank)
        gen = (lambda out, c0=c0, c1=c1: workloads.generate(key, col0=c0, ncols=c1 - c0, out=out))
        return dict(key=key, desc=f"{key}: 1x{cfg.cols} {cfg.dtype} single row, {cfg.desc}, "
                                  f"chunk-sharded over {world} GPU(s)",
                    rows=1, cols=c1 - c0, dtype=cfg.dtype, gen=gen, scaling="strong", mode="chunk",
                    elements_total=cfg.elements)
    if scaling == "strong":
        r0, r1 = tpd.row_range(cfg.rows, world, rank)
        gen = (lambda out, r0=r0, r1=r1: workloads.generate(key, row0=r0, nrows=r1 - r0, out=out))
        return dict(key=key, desc=f"{key}: {cfg.rows}x{cfg.cols} {cfg.dtype} total, {cfg.desc}, "
                                  f"rows sharded ({cfg.rows}/{world} per GPU)",
                    rows=r1 - r0, cols=cfg.cols, dtype=cfg.dtype, gen=gen, scaling="strong", mode="rows",
                    elements_total=cfg.elements)
    # weak: every rank processes one full batch of the config (rank r uses seed r; rank 0 = the config)
    gen = (lambda out, s=rank: workloads.generate(key, seed=s, out=out))
    return dict(key=key, desc=f"{key}: {cfg.rows}x{cfg.cols} {cfg.dtype} per GPU, {cfg.desc}, rows sharded",
                rows=cfg.rows, cols=cfg.cols, dtype=cfg.dtype, gen=gen, scaling="weak", mode="rows",
                elements_total=cfg.elements * world)


# ---------------------------------------------------------------- reference arm (oracle on CPU)

def run_reference(args, world, rank):
    if rank != 0:
        return
    import oracle
    import workloads
    spec = workload_spec(args.workload, 1, 0, args.scaling)
    kind = spec["dtype"]
    per_elem = BYTES_PER_ELEM[("two_pass", kind)]
    # one step = oracle softmax over S rows (or an n-element chunk of a single row)
    if spec["mode"] == "rows":
        probe = workloads.generate(args.workload, row0=0, nrows=1)
        oracle.softmax(probe)  # loads the library
        t0 = time.perf_counter()
        oracle.softmax(probe)
        t_row = time.perf_counter() - t0
        S = int(max(1, min(spec["rows"], round(args.ref_step_s / max(t_row, 1e-6)))))
        x = workloads.generate(args.workload, row0=0, nrows=S)
        sample = f"{S} of {spec['rows']} rows of {args.workload} per step"
    else:
        n = min(spec["cols"], 1 << 24)
        x = workloads.generate(args.workload, col0=0, ncols=n)
        t0 = time.perf_counter()
        oracle.softmax(x)
        t1 = time.perf_counter() - t0
        n = int(min(spec["cols"], max(1 << 16, n * args.ref_step_s / max(t1, 1e-6))))
        x = workloads.generate(args.workload, col0=0, ncols=n)
        sample = f"first {n} elements of the {args.workload} row per step"
    for _ in range(args.warmup):
        oracle.softmax(x)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.softmax(x)
    dt = (time.perf_counter() - t0) / args.steps
    elems = x.size
    value = per_elem * elems / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": spec["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": spec["desc"], "sample": sample, "bytes_per_element": per_elem},
            "elements_per_s": elems / dt,
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": oracle.threads(), "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, spec):
    """The oracle as it stands on this host's cores, bounded sample (~10-20 s of CPU work)."""
    import oracle
    import workloads
    per_elem = BYTES_PER_ELEM[("two_pass", spec["dtype"])]
    key = spec["key"]
    if spec["mode"] == "rows":
        x = workloads.generate(key, row0=0, nrows=1)
    else:
        x = workloads.generate(key, col0=0, ncols=min(spec["cols"], 1 << 22))
    t0 = time.perf_counter()
    oracle.softmax(x)
    t1 = time.perf_counter() - t0
    reps = int(max(1, min(200, args.cpu_budget_s / max(t1, 1e-6))))
    if spec["mode"] == "rows":
        S = min(spec["rows"], reps)
        x = workloads.generate(key, row0=0, nrows=S)
        sample = f"oracle softmax of {S} rows x {spec['cols']} of {key}"
    else:
        n = int(min(spec["cols"], x.size * reps))
        x = workloads.generate(key, col0=0, ncols=n)
        sample = f"oracle softmax of the first {n} elements of the {key} row"
    t0 = time.perf_counter()
    oracle.softmax(x)
    dt = time.perf_counter() - t0
    return {"value": per_elem * x.size / dt / 1e9, "unit": "GB/s", "cores": oracle.threads(), "kind": "oracle",
            "sample": sample, "elements_per_s": x.size / dt, "cpu_model": cpu_model()}


# ---------------------------------------------------------------- our arm

KERNEL_NAMES = {"stream": "tp::stream_kernel<{In},kTwoPass>", "cluster": "tp::rowcl_kernel<{In}>",
                "general": "tp::general_kernel<{In},kTwoPass>", "small": "tp::small_kernel<{In}>",
                "phase": "tp::rowph_kernel<{In},kTwoPass>", "resident": "tp::rowres_kernel<{In}>"}


def traffic_from_profiles(workload: str, kernel: str):
    """DRAM bytes per launch of this workload's kernel from the committed ncu capture, else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(workload)
    if d is None or d.get("kernel") != kernel:
        return None
    return d.get("dram_bytes_per_launch")


class Runner:
    """Timing harness shared by the headline workload and the rows-sharded lines."""

    def __init__(self, args, world, rank, local):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.args, self.world, self.rank, self.local = args, world, rank, local
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream(self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, step, K, W, sample_clocks=False, marks=None):
        """K back-to-back steps between events on the launching stream, max over ranks.
        marks: optional list that step() fills with (start, end) event pairs of the dominant
        kernel(s); their mean summed duration per step is returned as launch_ms."""
        torch = self.torch
        for _ in range(W):
            step()
        torch.cuda.synchronize(self.dev)
        sampler = None
        if sample_clocks:
            sampler = ClockSampler(self.local)
            sampler.start()
            t_end = time.time() + self.args.clock_window_s
            while time.time() < t_end:
                step()
                torch.cuda.synchronize(self.dev)
        self.barrier()
        torch.cuda.synchronize(self.dev)
        if marks is not None:
            marks.clear()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for i in range(K):
            evs[i][0].record(self.stream)
            step()
            evs[i][1].record(self.stream)
        e1.record(self.stream)
        torch.cuda.synchronize(self.dev)
        self.barrier()
        clocks = sampler.stop() if sampler else None
        total_ms = self.max_over_ranks(e0.elapsed_time(e1))
        if marks:
            launch_ms = sum(a.elapsed_time(b) for a, b in marks) / K
        else:
            launch_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
        return total_ms, launch_ms, clocks

    def timed_graph(self, step, K, W):
        """Launch-bound workloads: the K steps captured once into a CUDA graph (stream-ordered,
        allocation-free entry points), W warm-up steps eagerly and one warm-up replay, then ONE
        replay timed with events on the replaying stream; clocks sampled around replays."""
        torch = self.torch
        cs = torch.cuda.Stream(self.dev)
        cs.wait_stream(self.stream)
        with torch.cuda.stream(cs):
            for _ in range(W):
                step()
            torch.cuda.synchronize(self.dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for _ in range(K):
                    step()
            g.replay()
            torch.cuda.synchronize(self.dev)
            sampler = ClockSampler(self.local)
            sampler.start()
            t_end = time.time() + self.args.clock_window_s
            while time.time() < t_end:
                g.replay()
                torch.cuda.synchronize(self.dev)
            self.barrier()
            torch.cuda.synchronize(self.dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            g.replay()
            e1.record(cs)
            torch.cuda.synchronize(self.dev)
        self.barrier()
        clocks = sampler.stop()
        total_ms = self.max_over_ranks(e0.elapsed_time(e1))
        return total_ms, e0.elapsed_time(e1) / K, clocks

    # ------------------------------------------------------------ one workload
    def load(self, spec):
        """The rank's input, generated on the host (seeded, shard-invariant), pinned, in HBM."""
        torch = self.torch
        rows, cols, dtype = spec["rows"], spec["cols"], spec["dtype"]
        hx = torch.empty((rows, cols), dtype=torch.float32 if dtype == "f32" else torch.int16, pin_memory=True)
        hxn = hx.numpy()
        if dtype == "f32":
            spec["gen"](hxn)
        else:
            hxn[...] = spec["gen"](None).view(np.int16)
            hx = hx.view(torch.bfloat16)
        return hx, hx.to(self.dev)

    def measure(self, spec, headline: bool):
        import paper_2001_04438_b200 as tp
        from paper_2001_04438_b200 import dist as tpd
        torch, args, world = self.torch, self.args, self.world
        rows, cols, dtype = spec["rows"], spec["cols"], spec["dtype"]
        n_local = rows * cols
        hx, x = self.load(spec)
        y = torch.empty((rows, cols), dtype=torch.float32, device=self.dev)
        ws = tp.new_workspace(rows, max(cols, 1), self.dev)
        chunked = spec["mode"] == "chunk" and world > 1
        peer = tpd.PeerPairExchange(rows, self.dev) if chunked and args.exchange.startswith("nvlink") else None
        marks: list = []
        torch_ev = torch.cuda.Event

        def mark(fn):
            a, b = torch_ev(enable_timing=True), torch_ev(enable_timing=True)
            a.record(self.stream)
            r = fn()
            b.record(self.stream)
            marks.append((a, b))
            return r

        if chunked:
            pairs_ws = ws

            def step_two_pass():
                if peer is not None:
                    if args.exchange == "nvlink-fused":
                        ep = mark(lambda: peer.push_partial(x, pairs_ws))
                        mark(lambda: peer.finish(x, ep, out=y, workspace=pairs_ws))
                    else:
                        p = mark(lambda: tp.partial(x, workspace=pairs_ws))
                        allp = peer.exchange(p)
                        mark(lambda: tp.finish(x, allp, world, out=y, workspace=pairs_ws))
                else:
                    p = mark(lambda: tp.partial(x, workspace=pairs_ws))
                    allp = tpd.exchange_pairs(p)
                    mark(lambda: tp.finish(x, allp, world, out=y, workspace=pairs_ws))
            launches_per_step = 4 if args.exchange == "nvlink" else 2
        else:
            def step_two_pass():
                tp.softmax_ex(x, tp.ALGO_TWO_PASS, out=y, workspace=ws)
            launches_per_step = 1

        in_bytes = n_local * (4 if dtype == "f32" else 2)
        use_graph = args.graph == "on" or (args.graph == "auto" and in_bytes <= (64 << 20) and not chunked)
        if use_graph:
            total_ms, launch_ms, clocks = self.timed_graph(step_two_pass, args.steps, args.warmup)
        else:
            total_ms, launch_ms, clocks = self.timed(step_two_pass, args.steps, args.warmup,
                                                     sample_clocks=headline, marks=marks if chunked else None)
        plan = tp.last_plan()  # which kernel the timed launches ran
        if plan["kernel"] == "cluster" and plan["lookahead_rows"] > 0:
            launches_per_step += 1  # the tail rows' concurrent launch
        kernel_name = KERNEL_NAMES.get(plan["kernel"], plan["kernel"]).format(In="float" if dtype == "f32" else "uint16_t")
        if chunked:  # the partial's and the finish's kernels (one untimed call each, after timing)
            In = "float" if dtype == "f32" else "uint16_t"
            names = {"phase": "tp::rowph_kernel<{In},{A}>", "stream": "tp::stream_kernel<{In},{A}>"}
            tp.partial(x, workspace=pairs_ws)
            kp = tp.last_plan()["kernel"]
            kernel_name = (names.get(kp, kp).format(In=In, A="kPartial") + " + "
                           + names.get(plan["kernel"], plan["kernel"]).format(In=In, A="kFinish"))
            self.torch.cuda.synchronize(self.dev)
        if tp.watchdog_flags(ws, reset=True):
            raise RuntimeError("watchdog fired during the benchmark: results invalid")

        elems_total = spec["elements_total"]
        per_elem = BYTES_PER_ELEM[("two_pass", dtype)]
        ms_per_step = total_ms / args.steps
        value = per_elem * elems_total / (ms_per_step * 1e-3) / 1e9
        peak, peak_src = measured_peaks()
        achieved = per_elem * n_local / (launch_ms * 1e-3) / 1e9
        res = {
            "workload": spec["desc"], "value": value, "ms_per_step": ms_per_step,
            "rows_per_rank": rows, "cols_per_rank": cols, "elements_total": elems_total,
            "elements_per_s": elems_total / (ms_per_step * 1e-3), "bytes_per_element": per_elem,
            "pct_of_8TBs": value / world / NOMINAL_HBM_GBS,
            "timing": ("one CUDA-graph replay of the K steps (launch-bound workload)" if use_graph
                       else "K back-to-back steps"),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profiles(spec["key"], kernel_name),
                         "kernel": kernel_name, "plan": plan, "algorithmic_bytes_per_launch": per_elem * n_local,
                         "launch_ms_mean": launch_ms, "peak_source": peak_src,
                         "note": ("achieved = the paper's compulsory bytes (2 reads + 1 write per element) of this "
                                  "rank's elements / the kernel time per step (CUDA events on the launching stream"
                                  + ("; chunk-sharded: partial + finish, the all_gather excluded" if chunked else "")
                                  + "); traffic = DRAM bytes per launch from profiles/ (ncu), lower where "
                                  "re-reads hit L2 / shared memory, so frac can exceed 1")},
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clocks,
        }

        # three-pass comparators, same data, same protocol (outside the timed region above)
        three = {}
        if not args.no_three_pass:
            for nm, algo in (("recompute", tp.ALGO_RECOMPUTE), ("reload", tp.ALGO_RELOAD)):
                per_sched = {}
                if chunked:
                    tot, _, _ = self.timed(lambda a=algo: tpd.chunk_sharded_softmax3(x, a, out=y, workspace=ws),
                                           args.steps, args.warmup)
                    per_sched["sharded"] = {"ms_per_step": tot / args.steps, "kernel": "stream (3 phases, 2 all_gathers)"}
                else:
                    # each comparator on its default schedule and, where it applies, on the one-
                    # cluster-per-row schedule the Two-Pass uses; the faster one is the comparison
                    for sname, sched in (("default", tp.SCHED_AUTO), ("cluster", tp.SCHED_CLUSTER)):
                        fn = (self.timed_graph if use_graph else self.timed)
                        tot, _, _ = fn(lambda a=algo, sc=sched: tp.softmax_ex(x, a, out=y, workspace=ws, schedule=sc),
                                       args.steps, args.warmup)
                        kname = tp.last_plan()["kernel"]
                        if sname == "cluster" and kname != "cluster":
                            break  # the cluster schedule does not apply to this shape
                        per_sched[sname] = {"ms_per_step": tot / args.steps, "kernel": kname}
                best = min(per_sched.values(), key=lambda r: r["ms_per_step"])
                ms = best["ms_per_step"]
                three[nm] = {"ms_per_step": ms, "kernel": best["kernel"],
                             "schedules": {k: v["ms_per_step"] for k, v in per_sched.items()},
                             "GBps_own_cost_model": BYTES_PER_ELEM[(nm, dtype)] * elems_total / (ms * 1e-3) / 1e9,
                             "GBps_at_two_pass_bytes": value * ms_per_step / ms,
                             "two_pass_speedup": ms / ms_per_step}
            if plan["kernel"] == "cluster":  # the same Two-Pass on the grid-wide stream schedule
                fn = (self.timed_graph if use_graph else self.timed)
                tot, _, _ = fn(lambda: tp.softmax_ex(x, tp.ALGO_TWO_PASS, out=y, workspace=ws,
                                                     schedule=tp.SCHED_STREAM), args.steps, args.warmup)
                ms = tot / args.steps
                three["two_pass_stream_schedule"] = {"ms_per_step": ms,
                                                     "GBps": per_elem * elems_total / (ms * 1e-3) / 1e9,
                                                     "cluster_schedule_speedup": ms / ms_per_step}
        res["three_pass"] = three or None

        # end to end through the public API on host (pinned) buffers: H2D + kernels + D2H per step
        if headline and not args.no_e2e:
            hy = torch.empty((rows, cols), dtype=torch.float32, pin_memory=True)
            if chunked:
                pipe = tpd.HostChunkPipeline(cols, self.dev, dtype=x.dtype)
                run = (lambda: pipe.run(hx, hy))
                api = "dist.HostChunkPipeline (per rank: pipelined H2D, softmax_partial, NCCL all_gather, " \
                      "softmax_finish, D2H)"
            else:
                run = (lambda: tp.softmax_host(hx, hy))
                api = "softmax_f32_host / softmax_bf16_f32_host (C ABI, host buffers)"
            for _ in range(2):
                run()
            self.barrier()
            t0 = time.perf_counter()
            ke = max(3, min(args.steps, 10))
            for _ in range(ke):
                run()
                self.barrier()
            dt = self.max_over_ranks((time.perf_counter() - t0) / ke)
            res["e2e"] = {"value": per_elem * elems_total / dt / 1e9, "unit": "GB/s",
                          "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": int(n_local * 4),
                          "ms_per_step": dt * 1e3, "steps": ke, "api": api,
                          "note": "bytes per step are this rank's; the value is the whole job's"}
            if not chunked:
                # the same calls submitted asynchronously, two in flight (softmax_host_submit /
                # softmax_host_wait): each step still copies its input up and its output down,
                # one step's uploads overlapping the previous step's downloads
                try:
                    hys = [hy, torch.empty((rows, cols), dtype=torch.float32, pin_memory=True)]
                except RuntimeError as ex:  # host memory for a second pinned output
                    hys = None
                    res["e2e"]["pipelined_unavailable"] = str(ex)[:80]
                if hys is not None:
                    for t in [tp.softmax_host_submit(hx, hys[i]) for i in range(2)]:
                        tp.host_wait(t)
                    t0 = time.perf_counter()
                    tickets = []
                    for i in range(ke):
                        if i >= 2:
                            tp.host_wait(tickets[i - 2])
                        tickets.append(tp.softmax_host_submit(hx, hys[i % 2]))
                    for t in tickets[-2:]:
                        tp.host_wait(t)
                    dtp = self.max_over_ranks((time.perf_counter() - t0) / ke)
                    single = {k: res["e2e"][k] for k in ("value", "ms_per_step", "api")}
                    res["e2e"].update({"value": per_elem * elems_total / dtp / 1e9, "ms_per_step": dtp * 1e3,
                                       "api": "softmax_host_submit / softmax_host_wait (C ABI, host buffers, "
                                              "two calls in flight)",
                                       "single_call": single})
                    del hys
            del hy
        if peer is not None:
            peer.close()
        del x, y, ws, hx
        torch.cuda.empty_cache()
        return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--also", default="c4,c4b",
                    help="rows-sharded configurations measured beside the headline ('' = none)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="row configurations: strong = rows/N per rank (default), weak = a full batch per rank")
    ap.add_argument("--clock-window-s", type=float, default=1.0)
    ap.add_argument("--cpu-budget-s", type=float, default=8.0)
    ap.add_argument("--ref-step-s", type=float, default=1.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="time the K steps as one CUDA-graph replay (auto: launch-bound workloads, "
                         "<= 64 MB per rank, e.g. c1 / c2)")
    ap.add_argument("--no-three-pass", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "nvlink", "nvlink-fused"],
                    help="rank merge of chunk-sharded rows: NCCL all_gather or one-sided NVLink mailboxes")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and world == 1:
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                   "--master-port=29517", *sys.argv])
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    import workloads

    # development only (functional check of the N > 1 code paths on a one-GPU box; not a
    # measurement): TP_BENCH_ONE_DEVICE=1 puts every rank on cuda:0, TP_BENCH_BACKEND=gloo
    # replaces NCCL, which refuses two ranks on one device
    if os.environ.get("TP_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("TP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    if args.workload == "c5":  # M of the ties: one host scan on rank 0, broadcast (reading G16)
        v = [workloads.c5_tie_value() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(v, src=0)
        workloads.set_c5_tie_value(v[0])

    runner = Runner(args, world, rank, local)
    spec = workload_spec(args.workload, world, rank, args.scaling)
    head = runner.measure(spec, headline=True)
    also = {}
    for key in [k for k in args.also.split(",") if k and k != args.workload]:
        also[key] = runner.measure(workload_spec(key, world, rank, args.scaling), headline=False)
    cpu = cpu_baseline(args, spec) if (rank == 0 and world == 1) else None

    if rank == 0:
        chunked = spec["mode"] == "chunk" and world > 1
        line = {
            "metric": METRIC, "value": head["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": spec["scaling"], "vs_baseline": None, "dtype": spec["dtype"], "data": "synthetic",
            "config": {"workload": spec["desc"], "rows_per_rank": spec["rows"], "cols_per_rank": spec["cols"],
                       "elements_total": spec["elements_total"], "bytes_per_element": head["bytes_per_element"],
                       "l2": ("inputs larger than L2 (no flush): %.0f MB/rank > 126 MB"
                              % (spec["rows"] * spec["cols"] * (4 if spec["dtype"] == "f32" else 2) / 1e6)),
                       "timing": head["timing"],
                       "parallelism": ("rows sharded, no collective" if spec["mode"] == "rows" else
                                       ("one GPU, whole row" if world == 1 else
                                        "row chunk-sharded, one 8-byte (m,n) per rank exchanged by " +
                                        {"nvlink": "one-sided NVLink mailboxes (push / wait kernels)",
                                         "nvlink-fused": "one-sided NVLink mailboxes, pushed by the pass-1 kernel "
                                                         "and awaited by the pass-2 kernel"}.get(
                                            args.exchange, "NCCL all_gather")))},
            "elements_per_s": head["elements_per_s"],
            "pct_of_8TBs": head["pct_of_8TBs"],
            "roofline": head["roofline"],
            "three_pass": head["three_pass"],
            "rows_sharded": {k: {kk: vv for kk, vv in v.items() if kk not in ("clocks",)} for k, v in also.items()}
                            or None,
            "cpu_baseline": cpu,
            "e2e": head.get("e2e"),
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
        }
        if chunked:
            line["config"]["exchange"] = args.exchange
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
