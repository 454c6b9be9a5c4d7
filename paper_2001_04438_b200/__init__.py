"""Two-Pass softmax (Dukhan & Ablavatski, arXiv 2001.04438) on B200 — Python binding.

Thin ctypes marshalling over libtwopass.so (C ABI: include/twopass.h).  Every
step of the computation runs in the library's sm_100a kernels; this module only
passes device pointers, sizes and the current CUDA stream.  There is no CPU or
PyTorch fallback: if the library is missing or no GPU is present, calls raise.

    softmax(x)                   Alg. 3 SoftmaxTwoPass
    softmax3_recompute(x)        Alg. 1, PAPER.md:88-104   (in-house comparator)
    softmax3_reload(x)           Alg. 2, PAPER.md:108-128  (in-house comparator)
    partial(x) / finish(x, pairs, world)
                                 Alg. 3 pass 1 / pass 2 split for sharded rows
    softmax_host(hx, hy)         end-to-end call on host buffers
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# TP_LIBRARY: development override (an alternative in-tree build of the same library)
_SO = os.environ.get("TP_LIBRARY") or os.path.join(_PKG, "libtwopass.so")

TP_OK, TP_EINVAL, TP_ECUDA, TP_ENODEV, TP_EWATCHDOG = 0, 1, 2, 3, 4
ALGO_TWO_PASS, ALGO_RECOMPUTE, ALGO_RELOAD = 0, 2, 3
SCHED_AUTO, SCHED_STREAM, SCHED_HOLD, SCHED_CLUSTER, SCHED_SMALL, SCHED_PHASE, SCHED_RESIDENT = 0, 1, 2, 3, 4, 5, 6  # TP_SCHED_*
IN_F32, IN_BF16 = 0, 1

EXPORTS = [
    "softmax_f32", "softmax_bf16_f32", "softmax3_recompute_f32", "softmax3_reload_f32",
    "softmax3_recompute_bf16_f32", "softmax3_reload_bf16_f32", "softmax_f32_partial",
    "softmax_bf16_partial", "softmax_f32_finish", "softmax_bf16_f32_finish", "softmax_workspace_bytes",
    "softmax_ex", "softmax_partial_ex", "softmax_finish_ex", "softmax_partial_push_ex", "softmax_finish_mailbox_ex", "softmax_f32_host", "softmax_bf16_f32_host", "softmax_host_submit", "softmax_host_wait",
    "softmax_status_str", "softmax_last_cuda_error", "softmax_watchdog_flags", "softmax_last_plan", "tp_debug_op",
    "tp_bench_compute", "tp_set_profile_buffer", "tp_stream_baseline", "tp_read_probe", "tp_copy_probe", "tp_phase_only", "tp_exp_sweep", "tp_exp_fit",
    "softmax3_max_partial_ex", "softmax3_sum_partial_ex", "softmax3_finish_ex",
    "tp_mailbox_bytes", "tp_mailbox_pairs_offset", "tp_pairs_push", "tp_pairs_wait", "tp_ipc_get_handle", "tp_ipc_open", "tp_ipc_close",
]


class TwoPassError(RuntimeError):
    pass


class SoftmaxOpts(ctypes.Structure):
    _fields_ = [("grid_ctas", ctypes.c_int64), ("lookahead_rows", ctypes.c_int64),
                ("force_persistent", ctypes.c_int), ("disable_tma", ctypes.c_int),
                ("schedule", ctypes.c_int), ("cluster_size", ctypes.c_int)]


class SoftmaxPlan(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int), ("variant", ctypes.c_int), ("grid_ctas", ctypes.c_int64),
                ("cluster_size", ctypes.c_int), ("lookahead_rows", ctypes.c_int64), ("hold", ctypes.c_int)]


KERNEL_NAMES = {0: "none", 1: "general", 2: "stream", 3: "cluster", 4: "small", 5: "phase", 6: "resident"}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libtwopass.so (built by __graft_entry__.build() / paper_2001_04438_b200/build.py)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no fallback implementation)")
        L = ctypes.CDLL(_SO)
        vp, i64, ci, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
        for nm in ("softmax_f32", "softmax_bf16_f32", "softmax3_recompute_f32", "softmax3_reload_f32",
                   "softmax3_recompute_bf16_f32", "softmax3_reload_bf16_f32"):
            getattr(L, nm).argtypes = [vp, vp, i64, i64, vp]
        for nm in ("softmax_f32_partial", "softmax_bf16_partial"):
            getattr(L, nm).argtypes = [vp, i64, i64, vp, vp]
        for nm in ("softmax_f32_finish", "softmax_bf16_f32_finish"):
            getattr(L, nm).argtypes = [vp, vp, i64, i64, vp, ci, vp]
        L.softmax_workspace_bytes.argtypes = [i64, i64]
        L.softmax_workspace_bytes.restype = sz
        L.softmax_ex.argtypes = [ci, ci, vp, vp, i64, i64, vp, sz, ctypes.POINTER(SoftmaxOpts), vp]
        L.softmax_partial_ex.argtypes = [ci, vp, i64, i64, vp, vp, sz, ctypes.POINTER(SoftmaxOpts), vp]
        L.softmax_finish_ex.argtypes = [ci, vp, vp, i64, i64, vp, ci, vp, sz, ctypes.POINTER(SoftmaxOpts), vp]
        L.softmax_partial_push_ex.argtypes = [ci, vp, i64, i64, vp, ci, ci, ctypes.c_uint, vp, vp, sz,
                                              ctypes.POINTER(SoftmaxOpts), vp]
        L.softmax_finish_mailbox_ex.argtypes = [ci, vp, vp, i64, i64, vp, ci, ctypes.c_uint, ctypes.c_ulonglong,
                                                vp, sz, ctypes.POINTER(SoftmaxOpts), vp]
        L.softmax3_max_partial_ex.argtypes = [ci, vp, i64, i64, vp, vp, sz, vp]
        L.softmax3_sum_partial_ex.argtypes = [ci, ci, vp, vp, i64, i64, vp, ci, vp, vp, sz, vp]
        L.softmax3_finish_ex.argtypes = [ci, ci, vp, vp, i64, i64, vp, vp, ci, vp, sz, vp]
        L.softmax_f32_host.argtypes = [vp, vp, i64, i64]
        L.softmax_bf16_f32_host.argtypes = [vp, vp, i64, i64]
        L.softmax_host_submit.argtypes = [ctypes.c_int, vp, vp, i64, i64, ctypes.POINTER(ctypes.c_ulonglong)]
        L.softmax_host_wait.argtypes = [ctypes.c_ulonglong]
        L.softmax_status_str.argtypes = [ci]
        L.softmax_status_str.restype = ctypes.c_char_p
        L.tp_debug_op.argtypes = [ci, vp, vp, vp, vp, i64, vp]
        L.softmax_watchdog_flags.argtypes = [vp, ci]
        L.tp_set_profile_buffer.argtypes = [vp]
        L.tp_exp_fit.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_uint32, i64, ci, vp, vp, vp]
        L.tp_mailbox_bytes.argtypes = [ci, i64]
        L.tp_mailbox_bytes.restype = sz
        L.tp_mailbox_pairs_offset.argtypes = [ci, i64, ctypes.c_uint]
        L.tp_mailbox_pairs_offset.restype = sz
        L.tp_pairs_push.argtypes = [vp, i64, vp, ci, ci, ctypes.c_uint, vp]
        L.tp_pairs_wait.argtypes = [vp, ci, ctypes.c_uint, ctypes.c_uint64, vp]
        L.tp_ipc_get_handle.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
        L.tp_ipc_open.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
        L.tp_ipc_close.argtypes = [vp]
        L.tp_exp_sweep.argtypes = [ci, ctypes.c_uint32, i64, vp, vp, vp]
        L.tp_stream_baseline.argtypes = [ci, vp, vp, i64, ctypes.c_float, i64, vp]
        L.tp_read_probe.argtypes = [vp, i64, i64, ci, i64, vp, vp]
        L.tp_copy_probe.argtypes = [vp, vp, i64, i64, ci, i64, ci, vp]
        L.tp_phase_only.argtypes = [ci, ci, ci, vp, vp, i64, i64, vp, ctypes.c_size_t, vp]
        L.tp_bench_compute.argtypes = [ci, ci, i64, ci, vp, vp]
        L.softmax_last_plan.argtypes = [ctypes.POINTER(SoftmaxPlan)]
        _lib = L
    return _lib


def _check(status: int, what: str) -> None:
    if status != TP_OK:
        msg = lib().softmax_status_str(status).decode()
        if status == TP_ECUDA:
            msg += f" (cudaError {lib().softmax_last_cuda_error()})"
        raise TwoPassError(f"{what}: {msg}")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(x: torch.Tensor | None = None) -> int:
    """The current CUDA stream (of x's device) as a raw handle."""
    if _raw_stream is not None:
        return _raw_stream(x.get_device() if x is not None else torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def _in_dtype(x: torch.Tensor) -> int:
    if x.dtype == torch.float32:
        return IN_F32
    if x.dtype == torch.bfloat16:
        return IN_BF16
    raise TypeError(f"two-pass softmax takes float32 or bfloat16 logits, got {x.dtype}")


def _rows_cols(x: torch.Tensor) -> tuple[int, int]:
    if x.dim() == 0:
        raise ValueError("softmax of a 0-d tensor")
    cols = x.shape[-1]
    rows = x.numel() // cols if cols else 0
    return rows, cols


def _prep(x: torch.Tensor) -> torch.Tensor:
    if not x.is_cuda:
        raise ValueError("x must be a CUDA tensor (use softmax_host for host buffers)")
    return x if x.is_contiguous() else x.contiguous()


def _opts(grid_ctas: int = 0, lookahead_rows: int = 0, force_persistent: bool = False, disable_tma: bool = False,
          schedule: int = 0, cluster_size: int = 0):
    if not (grid_ctas or lookahead_rows or force_persistent or disable_tma or schedule or cluster_size):
        return None
    return ctypes.pointer(SoftmaxOpts(grid_ctas, lookahead_rows, int(force_persistent), int(disable_tma),
                                      int(schedule), int(cluster_size)))


def softmax_ex(x: torch.Tensor, algo: int = ALGO_TWO_PASS, out: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None, grid_ctas: int = 0, lookahead_rows: int = 0,
               force_persistent: bool = False, disable_tma: bool = False,
               schedule: int = 0, cluster_size: int = 0) -> torch.Tensor:
    """Row-wise softmax over the last dim; fp32 output.  See include/twopass.h."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    y = torch.empty(x.shape, dtype=torch.float32, device=x.device) if out is None else out
    if not (y.is_contiguous() and y.dtype == torch.float32 and y.shape == x.shape):
        raise ValueError("out must be a contiguous float32 tensor of x's shape")
    ws_ptr, ws_bytes = (None, 0) if workspace is None else (workspace.data_ptr(), workspace.numel() *
                                                             workspace.element_size())
    opts = None if not (grid_ctas or lookahead_rows or force_persistent or disable_tma or schedule or cluster_size) \
        else _opts(grid_ctas, lookahead_rows, force_persistent, disable_tma, schedule, cluster_size)
    st = lib().softmax_ex(algo, _in_dtype(x), x.data_ptr(), y.data_ptr(), rows, cols, ws_ptr, ws_bytes, opts,
                          _stream(x))
    if st:
        _check(st, "softmax")
    return y


def softmax(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Two-Pass softmax (Alg. 3) over the last dim of a CUDA float32/bfloat16 tensor."""
    return softmax_ex(x, ALGO_TWO_PASS, out)


def softmax3_recompute(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    return softmax_ex(x, ALGO_RECOMPUTE, out)


def softmax3_reload(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    return softmax_ex(x, ALGO_RELOAD, out)


def workspace_bytes(rows: int, cols: int) -> int:
    return int(lib().softmax_workspace_bytes(rows, cols))


def new_workspace(rows: int, cols: int, device=None) -> torch.Tensor:
    """Zero-filled caller-owned workspace for the _ex entry points."""
    return torch.zeros(max(workspace_bytes(rows, cols), 1), dtype=torch.uint8, device=device or "cuda")


def partial(x: torch.Tensor, out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
            grid_ctas: int = 0, schedule: int = 0) -> torch.Tensor:
    """Pass 1 of Alg. 3 over a chunk of each row -> [rows, 2] fp32 (m_sum, n_sum)."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    p = torch.empty((rows, 2), dtype=torch.float32, device=x.device) if out is None else out
    ws_ptr, ws_bytes = (None, 0) if workspace is None else (workspace.data_ptr(),
                                                             workspace.numel() * workspace.element_size())
    st = lib().softmax_partial_ex(_in_dtype(x), x.data_ptr(), rows, cols, p.data_ptr(), ws_ptr, ws_bytes,
                                  _opts(grid_ctas, schedule=schedule), _stream(x))
    _check(st, "partial")
    return p


def _ws(workspace: torch.Tensor | None):
    return (None, 0) if workspace is None else (workspace.data_ptr(), workspace.numel() * workspace.element_size())


def finish(x: torch.Tensor, pairs: torch.Tensor, world: int, out: torch.Tensor | None = None,
           grid_ctas: int = 0, workspace: torch.Tensor | None = None, schedule: int = 0) -> torch.Tensor:
    """Merge `world` partials per row (pairs: [world, rows, 2]) and run pass 2 on the local chunk.
    `workspace`: the one the chunk's partial() used (None: the internal one, as partial's None)."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    assert pairs.is_cuda and pairs.dtype == torch.float32 and pairs.is_contiguous()
    assert pairs.numel() == world * rows * 2
    y = torch.empty(x.shape, dtype=torch.float32, device=x.device) if out is None else out
    st = lib().softmax_finish_ex(_in_dtype(x), x.data_ptr(), y.data_ptr(), rows, cols, pairs.data_ptr(), world,
                                 *_ws(workspace), _opts(grid_ctas, schedule=schedule), _stream(x))
    _check(st, "finish")
    return y


# ---- sharded Three-Pass comparators (include/twopass.h softmax3_*_partial_ex / finish_ex)

def softmax3_max_partial(x: torch.Tensor, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Alg. 1/2 pass 1 over a chunk of each row -> [rows] fp32 maxima."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    out = torch.empty(rows, dtype=torch.float32, device=x.device)
    _check(lib().softmax3_max_partial_ex(_in_dtype(x), x.data_ptr(), rows, cols, out.data_ptr(), *_ws(workspace),
                                         _stream(x)), "softmax3_max_partial")
    return out


def softmax3_sum_partial(x: torch.Tensor, algo: int, maxes: torch.Tensor, out: torch.Tensor | None = None,
                         workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Pass 2 over the chunk with mu = max over the world's maxima ([world, rows]) -> [rows] sums;
    Reload also writes exp(x - mu) into `out` (allocated if None)."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    assert maxes.is_cuda and maxes.dtype == torch.float32 and maxes.is_contiguous() and maxes.numel() % rows == 0
    if algo == ALGO_RELOAD and out is None:
        out = torch.empty(x.shape, dtype=torch.float32, device=x.device)
    sums = torch.empty(rows, dtype=torch.float32, device=x.device)
    _check(lib().softmax3_sum_partial_ex(algo, _in_dtype(x), x.data_ptr(), None if out is None else out.data_ptr(),
                                        rows, cols, maxes.data_ptr(), maxes.numel() // rows, sums.data_ptr(),
                                        *_ws(workspace), _stream(x)), "softmax3_sum_partial")
    return sums


def softmax3_finish(x: torch.Tensor, algo: int, maxes: torch.Tensor, sums: torch.Tensor,
                    out: torch.Tensor | None = None, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Pass 3 over the chunk with mu, sigma merged from the world's partials ([world, rows] each)."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    assert maxes.numel() == sums.numel() and maxes.numel() % rows == 0
    y = torch.empty(x.shape, dtype=torch.float32, device=x.device) if out is None else out
    _check(lib().softmax3_finish_ex(algo, _in_dtype(x), x.data_ptr(), y.data_ptr(), rows, cols, maxes.data_ptr(),
                                    sums.data_ptr(), maxes.numel() // rows, *_ws(workspace), _stream(x)),
           "softmax3_finish")
    return y


def partial_push(x: torch.Tensor, peer_ptrs: torch.Tensor, rank: int, world: int, epoch: int,
                 pair_out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                 grid_ctas: int = 0) -> None:
    """Pass 1 over a chunk of each row; the kernel pushes the row pairs into slot `rank` of every
    mailbox (peer_ptrs: device int64 [world]) and releases `epoch` (softmax_partial_push_ex)."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    assert peer_ptrs.is_cuda and peer_ptrs.dtype == torch.int64 and peer_ptrs.numel() == world
    ws_ptr, ws_bytes = (None, 0) if workspace is None else (workspace.data_ptr(),
                                                             workspace.numel() * workspace.element_size())
    st = lib().softmax_partial_push_ex(_in_dtype(x), x.data_ptr(), rows, cols, peer_ptrs.data_ptr(), rank, world,
                                       epoch, None if pair_out is None else pair_out.data_ptr(), ws_ptr, ws_bytes,
                                       _opts(grid_ctas), _stream(x))
    _check(st, "partial_push")


def finish_mailbox(x: torch.Tensor, mailbox: torch.Tensor, world: int, epoch: int, timeout_ns: int,
                   out: torch.Tensor | None = None, grid_ctas: int = 0,
                   workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Await `epoch` in the local mailbox inside the kernel, merge its world pairs per row, pass 2
    (softmax_finish_mailbox_ex)."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    y = torch.empty(x.shape, dtype=torch.float32, device=x.device) if out is None else out
    st = lib().softmax_finish_mailbox_ex(_in_dtype(x), x.data_ptr(), y.data_ptr(), rows, cols, mailbox.data_ptr(),
                                         world, epoch, timeout_ns, *_ws(workspace), _opts(grid_ctas), _stream(x))
    _check(st, "finish_mailbox")
    return y


def phase_only(x: torch.Tensor, algo: int, phase: int, workspace: torch.Tensor,
               out: torch.Tensor | None = None) -> torch.Tensor | None:
    """Measurement hook (tp_phase_only): phase `phase` of `algo` alone; a later phase uses the
    statistics left in `workspace` by the previous full schedule=SCHED_STREAM call."""
    x = _prep(x)
    rows, cols = _rows_cols(x)
    y = out
    if y is None and not (algo == ALGO_TWO_PASS and phase == 0):
        y = torch.empty(x.shape, dtype=torch.float32, device=x.device)
    st = lib().tp_phase_only(algo, _in_dtype(x), phase, x.data_ptr(), None if y is None else y.data_ptr(), rows,
                             cols, workspace.data_ptr(), workspace.numel() * workspace.element_size(), _stream(x))
    _check(st, "phase_only")
    return y


def softmax_host(hx: torch.Tensor, hy: torch.Tensor | None = None) -> torch.Tensor:
    """End-to-end softmax of a HOST (ideally pinned) tensor into a host fp32 tensor (synchronous)."""
    assert not hx.is_cuda and hx.is_contiguous()
    rows, cols = _rows_cols(hx)
    if hy is None:
        hy = torch.empty(hx.shape, dtype=torch.float32, pin_memory=hx.is_pinned())
    assert not hy.is_cuda and hy.is_contiguous() and hy.dtype == torch.float32
    f = lib().softmax_f32_host if _in_dtype(hx) == IN_F32 else lib().softmax_bf16_f32_host
    _check(f(hx.data_ptr(), hy.data_ptr(), rows, cols), "softmax_host")
    return hy


def softmax_host_submit(hx: torch.Tensor, hy: torch.Tensor) -> int:
    """Asynchronous end-to-end softmax of a HOST tensor into a host fp32 tensor: returns a ticket
    for host_wait(); consecutive submissions overlap (include/twopass.h softmax_host_submit).
    hx and hy must stay alive and untouched until host_wait(ticket) returns."""
    assert not hx.is_cuda and hx.is_contiguous()
    assert not hy.is_cuda and hy.is_contiguous() and hy.dtype == torch.float32 and hy.shape == hx.shape
    rows, cols = _rows_cols(hx)
    t = ctypes.c_ulonglong(0)
    _check(lib().softmax_host_submit(_in_dtype(hx), hx.data_ptr(), hy.data_ptr(), rows, cols, ctypes.byref(t)),
           "softmax_host_submit")
    return t.value


def host_wait(ticket: int) -> None:
    _check(lib().softmax_host_wait(ticket), "softmax_host_wait")


def last_plan() -> dict:
    """What the last launch of this host thread ran (kernel, grid, cluster size, ...)."""
    p = SoftmaxPlan()
    _check(lib().softmax_last_plan(ctypes.byref(p)), "softmax_last_plan")
    return {"kernel": KERNEL_NAMES.get(p.kernel, str(p.kernel)), "variant": p.variant, "grid_ctas": p.grid_ctas,
            "cluster_size": p.cluster_size, "lookahead_rows": p.lookahead_rows, "hold": p.hold}


def watchdog_flags(workspace: torch.Tensor | None = None, reset: bool = True) -> int:
    """Watchdog bits of a workspace (None = internal); 0 means no pass-2 wait ever timed out."""
    return int(lib().softmax_watchdog_flags(None if workspace is None else workspace.data_ptr(), int(reset)))


def debug_op(what: int, a: torch.Tensor, b: torch.Tensor | None = None):
    """Unit-test hook (include/twopass.h tp_debug_op)."""
    a = _prep(a.float())
    count = a.numel() // 2 if what in (2, 8) else a.numel()
    o0 = torch.empty(count, dtype=torch.float32, device=a.device)
    o1 = torch.empty(count, dtype=torch.float32, device=a.device)
    bp = _prep(b.float()).data_ptr() if b is not None else None
    _check(lib().tp_debug_op(what, a.data_ptr(), bp, o0.data_ptr(), o1.data_ptr(), count, _stream()), "debug_op")
    return o0, o1
