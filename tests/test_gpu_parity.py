"""GPU parity of the Two-Pass softmax (and Three-Pass comparators) against the oracle.

Every test calls the CUDA path through the C ABI (paper_2001_04438_b200 ctypes
binding) and grades element by element with oracle.check (rel 2e-5 for oracle
outputs >= FLT_MIN, abs 1e-37 below; BASELINE.json north_star).
"""
import numpy as np
import pytest
import torch

import oracle
import workloads
from gpu_helpers import assert_parity, to_dev, to_host

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2001_04438_b200")

ALGOS = {
    "two_pass": tp.ALGO_TWO_PASS,
    "recompute": tp.ALGO_RECOMPUTE,
    "reload": tp.ALGO_RELOAD,
}


# ------------------------------------------------------------------ configurations 1-4 (full size)

@pytest.mark.parametrize("algo", list(ALGOS))
@pytest.mark.parametrize("key", ["c1", "c2", "c3"])
def test_config_parity(key, algo):
    x = workloads.generate(key)
    y = to_host(tp.softmax_ex(to_dev(x), ALGOS[algo]))
    r = assert_parity(x, y, f"{key}/{algo}")
    assert r.n_rel > 0
    assert abs(r.y_sum - x.shape[0]) <= 2e-5 * x.shape[0]


@pytest.mark.parametrize("algo", list(ALGOS))
@pytest.mark.parametrize("key", ["c4", "c4b"])
def test_config4_parity(key, algo):
    x = workloads.generate(key)
    y = to_host(tp.softmax_ex(to_dev(x), ALGOS[algo]))
    assert_parity(x, y, f"{key}/{algo}")


def test_config1_naive_overflows_but_two_pass_is_finite():
    # PAPER.md:76 / SPEC.md:407: a naive fp32 softmax of config 1 is inf/NaN
    x = workloads.generate("c1")
    xt = to_dev(x)
    naive = torch.exp(xt) / torch.exp(xt).sum()
    assert not bool(torch.isfinite(naive).all())
    y = tp.softmax(xt)
    assert bool(torch.isfinite(y).all())


# ------------------------------------------------------------------ config 5 (2^31 elements), every output

@pytest.mark.slow
def test_config5_full_size_every_output():
    # all 2^31 outputs graded against the oracle with the full row's statistics (copied back and
    # graded in 2^26-element chunks), then the chunk-sharded path at W = 8 (emulated on this GPU:
    # partials of the 8 block-aligned chunks, the gathered pairs, 8 finishes) bitwise equal to the
    # one-GPU output at full size (pin P9)
    cfg = workloads.CONFIGS["c5"]
    n = cfg.cols
    host = torch.empty((1, n), dtype=torch.float32, pin_memory=True)
    x = host.numpy()
    workloads.generate("c5", out=x)
    xd = host.cuda(non_blocking=True)
    y = tp.softmax(xd)
    torch.cuda.synchronize()
    stats = oracle.row_stats(x[0])                     # full-row oracle statistics
    ybuf = torch.empty((1 << 26,), dtype=torch.float32, pin_memory=True)
    res = None
    for c0 in range(0, n, 1 << 26):
        c1 = min(n, c0 + (1 << 26))
        ybuf[: c1 - c0].copy_(y[0, c0:c1])
        r = oracle.check(x[0, c0:c1], ybuf[: c1 - c0].numpy(), stats)
        res = r if res is None else res.merge(r, offset=c0)
    assert res.ok, (res.n_bad, res.first_bad, res.max_rel, res.max_abs)
    assert res.n_rel + res.n_abs == n
    assert res.n_rel > 20_000_000                      # the ~1% ties sit in the relative branch
    assert abs(res.y_sum - 1.0) <= 2e-5
    ties = np.nonzero(x[0] == x[0].max())[0]
    yt = y[0, torch.from_numpy(ties[:1_000_000]).cuda()]
    assert float(yt.max()) == float(yt.min())          # equal inputs, equal outputs
    # W = 8 chunk-sharded, bitwise
    from paper_2001_04438_b200 import dist as tpd
    world = 8
    spans = [tpd.chunk_range(n, world, r) for r in range(world)]
    wss = [tp.new_workspace(1, b - a) for a, b in spans]
    pairs = torch.stack([tp.partial(xd[:, a:b], workspace=w) for (a, b), w in zip(spans, wss)]).contiguous()
    y8 = torch.empty_like(y)
    for (a, b), w in zip(spans, wss):  # one row: the column slices are contiguous
        tp.finish(xd[:, a:b], pairs, world, out=y8[:, a:b], workspace=w)
    assert torch.equal(y8, y)
    del xd, y, y8
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ ragged shapes and dtypes

RAGGED = [(1, 1), (1, 2), (3, 3), (2, 5), (4, 17), (1, 1000), (7, 4095), (3, 4096), (5, 4097),
          (2, 16383), (2, 16384), (2, 16385), (3, 32773), (1, 65537), (2, 200003), (1, 16384 * 64 + 1),
          (1, 16384 * 65), (3, 16384 * 130 + 7), (300, 33)]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", RAGGED)
def test_ragged_two_pass(rows, cols, dtype):
    x = workloads.ragged_case(rows, cols, -300.0, 300.0, seed=rows, stream=cols)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    y = to_host(tp.softmax(to_dev(x)))
    assert_parity(x, y, f"{rows}x{cols}/{dtype}")


@pytest.mark.parametrize("algo", ["recompute", "reload"])
@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 17), (2, 16385), (1, 16384 * 65 + 3), (5, 4097)])
def test_ragged_three_pass(rows, cols, algo):
    x = workloads.ragged_case(rows, cols, -300.0, 300.0, seed=rows, stream=cols + 1)
    y = to_host(tp.softmax_ex(to_dev(x), ALGOS[algo]))
    assert_parity(x, y, f"{rows}x{cols}/{algo}")


@pytest.mark.parametrize("cols", [1000, 4097, 50001])
def test_misaligned_rows(cols):
    # a view starting one element into the buffer: no 16-byte alignment anywhere
    base = workloads.ragged_case(1, 3 * cols + 1, -50, 50, seed=9, stream=cols)[0]
    xd = to_dev(base)[1:].view(3, cols)
    assert xd.data_ptr() % 16 != 0
    y = to_host(tp.softmax(xd))
    assert_parity(base[1:].reshape(3, cols), y, "misaligned")
    # and the aligned copy gives the same bits (per-thread assignment does not depend on alignment)
    y2 = to_host(tp.softmax(xd.contiguous().clone()))
    assert np.array_equal(y, y2)


# ------------------------------------------------------------------ edge cases and contracts

def test_empty_and_invalid_inputs():
    L = tp.lib()
    x = torch.zeros(4, device="cuda")
    y = torch.zeros(4, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert L.softmax_f32(x.data_ptr(), y.data_ptr(), 0, 4, s) == tp.TP_EINVAL
    assert L.softmax_f32(x.data_ptr(), y.data_ptr(), 1, 0, s) == tp.TP_EINVAL
    assert L.softmax_f32(None, y.data_ptr(), 1, 4, s) == tp.TP_EINVAL
    assert L.softmax_f32(x.data_ptr(), x.data_ptr() + 4, 1, 3, s) == tp.TP_EINVAL   # partial overlap
    assert L.softmax_f32_finish(x.data_ptr(), y.data_ptr(), 1, 4, x.data_ptr(), 0, s) == tp.TP_EINVAL
    with pytest.raises(tp.TwoPassError):
        tp.softmax(torch.zeros(0, 5, device="cuda"))


@pytest.mark.parametrize("cols", [1000, 40000])
def test_in_place(cols):
    x = workloads.ragged_case(3, cols, -90, 90, seed=1, stream=2)
    xd = to_dev(x)
    tp.softmax(xd, out=xd)
    assert_parity(x, to_host(xd), "in-place")


@pytest.mark.parametrize("n", [1000, 32768, 1 << 20, 1 << 24])
def test_constant_zero_row_is_exactly_rn32_one_over_n(n):
    # P10: m_i = 1, n_i = 0, m_sum = N exactly, lambda = RN32(1/N) -> every output == RN32(1/N)
    y = to_host(tp.softmax(torch.zeros(1, n, device="cuda")))
    assert np.all(y == np.float32(1.0 / n))


def test_constant_nonzero_row():
    for c in [88.0, -1e4, 1e4, 3.25]:
        x = np.full((2, 70000), c, np.float32)
        assert_parity(x, to_host(tp.softmax(to_dev(x))), f"const {c}")


def test_extreme_magnitudes_stay_finite():
    x = np.float32([[1e4, -1e4, 0.0, 1e4], [3.4e38, -3.4e38, 0.0, 1.0], [-3.4e38, -3.4e38, -3.4e38, -3.4e38]])
    y = to_host(tp.softmax(to_dev(x)))
    assert np.all(np.isfinite(y)) and np.all(y >= 0)
    assert_parity(x[:1], y[:1], "±1e4")
    assert np.allclose(y.sum(1), 1.0, atol=2e-5)


def test_flush_boundary_rows():
    # reading G9 / SURVEY M11: two-element rows [x_max, x_max - d] with d just around the
    # FLT_MIN boundary of the smaller output; lambda' = 0.5 / m_sum keeps those outputs exact
    xm = workloads.uniform(400, -1e4, 1e4, seed=21, stream=1).astype(np.float32)
    rows = []
    for d in np.arange(87.30, 87.40, 0.0025):
        rows.append(np.stack([xm, (xm - np.float32(d)).astype(np.float32)], 1))
    x = np.concatenate(rows).astype(np.float32)
    y = to_host(tp.softmax(to_dev(x)))
    r = assert_parity(x, y, "flush boundary")
    assert r.n_rel > 0 and r.n_abs > 0


def test_integer_shift_invariance_within_tolerance():
    rng = np.random.default_rng(3)
    x = rng.integers(-2000, 2000, size=(4, 30000)).astype(np.float32)
    y0 = to_host(tp.softmax(to_dev(x)))
    for c in [1.0, -777.0, 4096.0]:
        xc = (x + np.float32(c)).astype(np.float32)
        yc = to_host(tp.softmax(to_dev(xc)))
        assert_parity(xc, yc, "shift")
        big = y0 > 1e-30
        assert np.max(np.abs(yc[big] - y0[big]) / y0[big]) <= 4e-5


# ------------------------------------------------------------------ determinism (reading G8, pin P9)

def test_bitwise_deterministic_across_grid_and_lookahead():
    x = workloads.ragged_case(9, 16384 * 5 + 11, -500, 500, seed=4, stream=4)
    xd = to_dev(x)
    ref = to_host(tp.softmax(xd))
    assert np.array_equal(ref, to_host(tp.softmax(xd)))
    for g, la in [(1, 0), (7, 1), (148, 2), (1000, 0), (37, 9)]:
        assert np.array_equal(ref, to_host(tp.softmax_ex(xd, grid_ctas=g, lookahead_rows=la))), (g, la)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", [(3, 1000), (2, 16384 * 3 + 8), (1, 16384 * 70)])
def test_tma_and_global_load_paths_agree_bitwise(rows, cols, dtype):
    x = workloads.ragged_case(rows, cols, -400, 400, seed=3, stream=cols)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    for algo in ALGOS.values():
        a = to_host(tp.softmax_ex(xd, algo))
        b = to_host(tp.softmax_ex(xd, algo, disable_tma=True))
        assert np.array_equal(a, b), algo


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", [(64, 32768), (9, 16384 * 5 + 12), (40, 800000)])
def test_hold_and_reread_schedules_agree_bitwise(rows, cols, dtype):
    # hold: blocks stay in shared memory between the passes; re-read: pass 2 reloads them
    x = workloads.ragged_case(rows, cols, -500, 500, seed=6, stream=cols)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    a = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_HOLD))
    b = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    assert np.array_equal(a, b)
    if rows * cols <= 2_000_000:
        assert_parity(x, a, "hold")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", [(64, 32768), (5, 16384 + 4), (9, 16384 * 5 + 12), (40, 800000),
                                       (3, 16384 * 64), (2, 16384 * 100 + 8), (2, 16384 * 256),
                                       (1, 16384 * 257), (300, 16384 * 2 + 100)])
def test_cluster_schedule_agrees_bitwise_with_stream(rows, cols, dtype):
    # cluster: one thread-block cluster per row, block values exchanged through DSMEM, pass 2
    # from shared memory / L2 (tp_rowcl.cu); stream: the row spread over the persistent grid.
    # Same canonical trees (reading G8), so the outputs must be bit-identical; 2..256 blocks
    # per row use the cluster kernel (nb = 257 falls back to the stream kernel).
    x = workloads.ragged_case(rows, cols, -500, 500, seed=8, stream=cols + rows)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    for cl in [0, 1, 2, 4, 8, 16]:
        y = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_CLUSTER, cluster_size=cl))
        assert tp.watchdog_flags() == 0
        assert np.array_equal(ref, y), (cl, rows, cols)
    assert np.array_equal(ref, to_host(tp.softmax(xd)))
    if rows * cols <= 3_000_000:
        assert_parity(x, ref, "cluster")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_cluster_schedule_many_short_rows(dtype):
    # thousands of rows of 2-3 blocks: every cluster loops over many rows (row parity buffers,
    # epoch-free barriers), shares of 1-2 blocks per CTA
    x = workloads.ragged_case(3000, 16384 * 2 + 1000, -80, 80, seed=13, stream=13)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    for cl in [0, 2, 3 - 1]:
        y = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_CLUSTER, cluster_size=cl))
        assert tp.watchdog_flags() == 0
        assert np.array_equal(ref, y), cl
    assert_parity(x[:64], ref[:64], "many short rows")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", [(1, 1000), (7, 16384), (64, 32768), (3, 16384 * 3), (5, 16384 * 2 + 36),
                                       (400, 16384 * 2 + 4)])
def test_small_schedule_agrees_bitwise(rows, cols, dtype):
    # one CTA per row of <= 3 blocks, row staged in shared memory (tp_small.cu); 400 rows loop
    x = workloads.ragged_case(rows, cols, -300, 300, seed=14, stream=rows + cols)
    x[0, 3] = 4.0e7 if rows > 1 else x[0, 3]       # one out-of-domain block (clamped path)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    y = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_SMALL))
    if cols % (8 if dtype == "bf16" else 4) == 0:       # 16-byte rows; others take the general kernel
        assert tp.last_plan()["kernel"] == "small"
    assert np.array_equal(ref, y)
    # 1..3 CTAs per row (a cluster sharing block values through DSMEM), and few clusters
    # looping over the rows: the same bits
    for cl, grid in ((1, 0), (2, 0), (3, 0), (2, 6), (3, 3)):
        yc = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_SMALL, cluster_size=cl, grid_ctas=grid))
        assert np.array_equal(ref, yc), (cl, grid)
    # the Three-Pass comparators on the same staging: bitwise equal to their stream-kernel runs
    for algo in ("recompute", "reload"):
        ref3 = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_STREAM))
        for cl in (0, 1, 3):
            y3 = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_SMALL, cluster_size=cl))
            assert np.array_equal(ref3, y3), (algo, cl)
        if rows * cols <= 3_000_000 and rows > 1:
            assert_parity(x[1:], ref3[1:], f"small {algo}")
    if rows * cols <= 3_000_000 and rows > 1:
        assert_parity(x[1:], y[1:], "small")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", [(5, 16384 * 4), (3, 16384 * 64), (40, 16384 * 7 + 8), (300, 16384 * 5 + 4000),
                                       (24, 16384 * 49 + 5000)])
def test_resident_schedule_agrees_bitwise(rows, cols, dtype):
    # a group of CTAs per row stages its whole share, exchanges block values through the
    # workspace tickets, pass 2 on the staged blocks (tp_rowres.cu): the same canonical trees as
    # the stream kernel, so the same bits; forced group sizes and capped grids make groups loop
    # over many rows (ticket reuse per row, stage refills across rows); clamped blocks (G11)
    x = workloads.ragged_case(rows, cols, -400, 400, seed=21, stream=rows + cols)
    x[0, 5] = 4.0e7
    x[rows - 1, cols - 3] = -2.0e9
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ws = tp.new_workspace(rows, cols)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM, workspace=ws))
    nb = -(-cols // 16384)
    bmax = 3 if dtype == "bf16" else 1
    gmin = -(-nb // bmax)
    y = to_host(tp.softmax_ex(xd, workspace=ws))  # AUTO: bf16 rows of one block per CTA take it
    assert np.array_equal(ref, y)
    if dtype == "bf16" and rows >= 2 * (148 // nb):
        assert tp.last_plan()["kernel"] == "resident"
    ran = 0
    for g, grid in ((0, 0), (gmin, 0), (min(nb, gmin + 1), 0), (gmin, 2 * gmin), (nb, 0), (gmin, gmin)):
        for rep in range(2):  # the same workspace twice: tickets left at zero by each launch
            y = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_RESIDENT, cluster_size=g, grid_ctas=grid, workspace=ws))
            assert tp.watchdog_flags(ws) == 0
            assert np.array_equal(ref, y), (g, grid, rep)
        ran += tp.last_plan()["kernel"] == "resident"
    assert ran >= 5
    # a stream launch on the same workspace afterwards (control region shared): still the same
    assert np.array_equal(ref, to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM, workspace=ws)))
    # the Three-Pass comparators on the same schedule: bitwise equal to their stream-kernel runs
    for algo in ("recompute", "reload"):
        ref3 = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_STREAM, workspace=ws))
        for g, grid in ((0, 0), (nb, 0), (gmin, 0), (gmin, gmin)):
            y3 = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_RESIDENT, cluster_size=g, grid_ctas=grid,
                                       workspace=ws))
            assert tp.watchdog_flags(ws) == 0
            assert np.array_equal(ref3, y3), (algo, g, grid)
        if rows * cols <= 3_000_000:
            assert_parity(x[1:], ref3[1:], f"resident {algo}")
    if rows * cols <= 3_000_000:
        assert_parity(x, ref, "resident")
    else:
        assert_parity(x[:2], ref[:2], "resident")


def test_resident_schedule_graph_capture_and_streams():
    # the resident-row launch inside a CUDA graph, replayed; and two workspaces on two streams
    x = workloads.to_bf16(workloads.ragged_case(64, 16384 * 20 + 304, -300, 300, seed=22, stream=22))
    xd = to_dev(x)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    ws = tp.new_workspace(*x.shape)
    y = torch.empty(x.shape, dtype=torch.float32, device="cuda")
    tp.softmax_ex(xd, out=y, workspace=ws)
    assert tp.last_plan()["kernel"] == "resident"
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        tp.softmax_ex(xd, out=y, workspace=ws)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tp.softmax_ex(xd, out=y, workspace=ws)
    for _ in range(3):
        y.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(ref, to_host(y))
    assert tp.watchdog_flags(ws) == 0
    assert_parity(x[:3], ref[:3], "resident graph")


def test_cluster_schedule_clamped_blocks_and_small_grids():
    # out-of-domain blocks (reading G11) inside multi-block rows: the per-warp clamp masks stay
    # local to the CTA that ran pass 1; a capped grid makes clusters loop over many rows
    x = workloads.ragged_case(24, 16384 * 6 + 40, -50, 50, seed=9, stream=9)
    x[1, 100] = 3.0e7
    x[5, 16384 * 3 + 7] = -1.0e9
    x[7, :] = -5.0e6
    xd = to_dev(x)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    for cl, g in [(2, 2), (4, 8), (1, 1), (8, 0)]:
        y = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_CLUSTER, cluster_size=cl, grid_ctas=g))
        assert np.array_equal(ref, y), (cl, g)
    assert np.isfinite(ref).all()


def test_out_of_domain_blocks_take_the_clamped_path():
    # a row with one huge element, a row entirely below -2^21, a row with +-inf/NaN-free extremes:
    # outputs finite, non-negative, summing to 1; in-domain rows unaffected (reading G11)
    x = workloads.ragged_case(4, 40000, -50, 50, seed=1, stream=77)
    x[0, 12345] = 1e30
    x[1, :] = -5e6
    x[1, 777] = -4e6
    x[2, 100] = 3e6
    y = to_host(tp.softmax(to_dev(x)))
    assert np.all(np.isfinite(y)) and np.all(y >= 0)
    assert np.allclose(y.sum(1), 1.0, atol=2e-5)
    assert abs(y[0, 12345] - 1.0) <= 2e-7 and abs(y[2, 100] - 1.0) <= 2e-7
    assert_parity(x[3:], y[3:], "in-domain row")


def test_rowblock_and_persistent_paths_agree_bitwise():
    for cols in [1, 1000, 16384]:
        xd = to_dev(workloads.ragged_case(5, cols, -100, 100, seed=5, stream=cols))
        a = to_host(tp.softmax(xd))
        b = to_host(tp.softmax_ex(xd, force_persistent=True))
        assert np.array_equal(a, b), cols


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_partial_finish_world_invariance(dtype):
    # one long row split into W equal block-aligned chunks: partial per chunk, finish with all
    # W pairs -> bit-identical to the single-call result for W in {1, 2, 4, 8} (pin P9)
    n = 16384 * 256
    x = workloads.uniform(n, -1e4, 1e4, seed=8, stream=8).reshape(1, n)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ref = to_host(tp.softmax(xd))
    assert_parity(x, ref, "single call")
    for W in [1, 2, 4, 8]:
        c = n // W
        chunks = [xd[:, w * c:(w + 1) * c].contiguous() for w in range(W)]
        pairs = torch.stack([tp.partial(ch) for ch in chunks])        # [W, rows, 2]
        ys = [tp.finish(ch, pairs, W) for ch in chunks]
        y = to_host(torch.cat(ys, dim=1))
        assert np.array_equal(y, ref), W


def test_partial_pair_represents_row_sum():
    # the chunk pair is (m_sum, n_sum) with m_sum 2^n_sum = sum_i e^{x_i}
    x = workloads.ragged_case(3, 100000, -2000, 2000, seed=2, stream=6)
    p = to_host(tp.partial(to_dev(x)))
    for r in range(3):
        mu, S = oracle.row_stats(x[r])
        # log of the represented sum vs log of mu-shifted oracle sum: n ln2 + ln m = mu + ln S
        lhs = p[r, 1] * np.log(2.0) + np.log(p[r, 0])
        rhs = mu + float(np.log(S))
        assert abs(lhs - rhs) <= 2e-5 * max(1.0, abs(rhs)) + 2e-5


# ------------------------------------------------------------------ end-to-end host path

@pytest.mark.parametrize("key", ["c2", "c3"])
def test_host_pipeline_matches_device_path(key):
    x = workloads.generate(key)
    hx = torch.from_numpy(x).pin_memory()
    hy = tp.softmax_host(hx)
    ref = to_host(tp.softmax(to_dev(x)))
    assert np.array_equal(hy.numpy(), ref)


def test_host_pipeline_slab_ramp_bitwise():
    # 200 rows of C4 bf16 (320 MB in): a doubling ramp of small slabs at both ends, full slabs
    # between, alternating streams; every slab's launch gives the device path's bits (fp32 too)
    x = workloads.generate("c4b", 0, 200)
    hx = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory()
    hy = tp.softmax_host(hx)
    ref = to_host(tp.softmax(hx.cuda()))
    assert np.array_equal(hy.numpy(), ref)
    x = workloads.generate("c4", 0, 100)
    hy = tp.softmax_host(torch.from_numpy(x).pin_memory()).numpy()
    ref = to_host(tp.softmax(to_dev(x)))
    if not np.array_equal(hy, ref):  # say where, and which side the oracle disowns
        rows = np.unique(np.nonzero(hy != ref)[0])
        sides = []
        for name, y in (("host", hy), ("device", ref)):
            try:
                assert_parity(x[rows[:4]], y[rows[:4]])
            except AssertionError:
                sides.append(name)
        raise AssertionError(f"host and device paths differ in rows {rows[:16].tolist()} ({len(rows)} rows); "
                             f"outside the oracle tolerance: {sides or 'neither'}; watchdog {tp.watchdog_flags()}")


def test_host_submit_overlapping_calls_bitwise():
    # the asynchronous host-buffer call: calls in flight on the two staging slots (and a third
    # queued behind the first), each result the synchronous call's bits; single long row (chunked
    # path) and row slabs (bf16 and fp32)
    cases = [workloads.generate("c3")[:, : 1 << 24], workloads.generate("c4", 0, 40)]
    xb = workloads.generate("c4b", 0, 30)
    hxs = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in cases]
    hxs.append(torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).pin_memory())
    for hx in hxs:
        ref = tp.softmax_host(hx)
        hys = [torch.empty(hx.shape, dtype=torch.float32).pin_memory() for _ in range(3)]
        tickets = [tp.softmax_host_submit(hx, hy) for hy in hys]
        for t in reversed(tickets):
            tp.host_wait(t)
        for hy in hys:
            assert torch.equal(hy, ref)
    with pytest.raises(tp.TwoPassError):
        tp.host_wait(0)
    with pytest.raises(tp.TwoPassError):
        tp.host_wait(tickets[-1] + 1)  # not submitted yet


def test_host_pipeline_bf16_and_multi_slab():
    x = workloads.generate("c4b", 0, 40)
    hx = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory()
    hy = tp.softmax_host(hx)
    assert_parity(x, hy.numpy(), "host bf16")


def test_auto_tuner_picks_a_candidate_and_keeps_results_bitwise(tmp_path):
    # NEXT-3 meta-parameter tuner: every candidate gives the same bits, so the tuned launch must too
    from paper_2001_04438_b200 import tune
    x = workloads.ragged_case(24, 16384 * 7 + 20, -300, 300, seed=12, stream=12)
    xd = to_dev(x)
    cache = str(tmp_path / "tune.json")
    best = tune.tune(xd, reps=2, cache_path=cache)
    assert best in tune.candidates(24, x.shape[1])
    assert tune.tune(xd, cache_path=cache) == best            # cached
    y = to_host(tune.softmax_tuned(xd, cache_path=cache))
    assert np.array_equal(y, to_host(tp.softmax(xd)))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("algo", list(ALGOS))
@pytest.mark.parametrize("grid", [1, 4, 0])
def test_fresh_workspace_small_grids_repeated(algo, dtype, grid):
    # regression: the stream kernel's producer once stalled after one round of stages for bf16
    # Three-Pass Recompute on a fresh workspace (stage bookkeeping in local arrays); every
    # algorithm, dtype and grid size on a fresh workspace, three launches, watchdog clear
    x = workloads.ragged_case(3, 16384 * 10 + 96, -200, 200, seed=15, stream=grid)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ws = tp.new_workspace(*x.shape)
    ys = []
    for _ in range(3):
        ys.append(to_host(tp.softmax_ex(xd, ALGOS[algo], workspace=ws, grid_ctas=grid, schedule=tp.SCHED_STREAM)))
        assert tp.watchdog_flags(ws) == 0
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2])
    assert_parity(x, ys[0], f"{algo}/{dtype}/grid {grid}")


def test_cuda_graph_capture_replays_bitwise():
    # the entry points are stream-ordered, allocation-free and host-sync-free: capturable in a
    # CUDA graph, including the cluster launch with its concurrent tail launch (fork / join events)
    x = workloads.ragged_case(256, 16384 * 49 + 5000, -300, 300, seed=16, stream=16)
    xd = to_dev(x)
    y = torch.empty_like(xd)
    ws = tp.new_workspace(*x.shape)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    tp.softmax_ex(xd, out=y, workspace=ws)
    plan = tp.last_plan()
    assert plan["kernel"] == "cluster" and plan["lookahead_rows"] > 0   # cluster launch + tail launch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        tp.softmax_ex(xd, out=y, workspace=ws)      # warm-up (lazy init outside the capture)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tp.softmax_ex(xd, out=y, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        y.zero_()
        g.replay()
        assert np.array_equal(to_host(y), ref)
    assert tp.watchdog_flags(ws) == 0


def test_concurrent_streams_with_own_workspaces():
    # two launches on two streams at once, each with its own workspace (include/twopass.h)
    xa = to_dev(workloads.ragged_case(200, 16384 * 6 + 8, -100, 100, seed=17, stream=1))
    xb = to_dev(workloads.ragged_case(3, 16384 * 300, -100, 100, seed=17, stream=2))
    ra = to_host(tp.softmax_ex(xa, schedule=tp.SCHED_STREAM))
    rb = to_host(tp.softmax_ex(xb, schedule=tp.SCHED_STREAM))
    wa, wb = tp.new_workspace(*xa.shape), tp.new_workspace(*xb.shape)
    ya, yb = torch.empty_like(xa), torch.empty_like(xb)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    sa.wait_stream(torch.cuda.current_stream())
    sb.wait_stream(torch.cuda.current_stream())
    for _ in range(3):
        with torch.cuda.stream(sa):
            tp.softmax_ex(xa, out=ya, workspace=wa)
        with torch.cuda.stream(sb):
            tp.softmax_ex(xb, out=yb, workspace=wb)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(ya), ra) and np.array_equal(to_host(yb), rb)
    assert tp.watchdog_flags(wa) == 0 and tp.watchdog_flags(wb) == 0


def test_workspace_reused_across_shapes_and_schedules():
    # one workspace, alternating shapes (control regions re-zeroed on shape change) and
    # schedules (cluster with tail split, stream, small), results stay bitwise stable
    shapes = [(256, 16384 * 49 + 5000), (40, 16384 * 3), (256, 16384 * 49 + 5000), (7, 16384 * 2 + 40)]
    ws = tp.new_workspace(256, 16384 * 49 + 5000)
    refs = {}
    for it in range(2):
        for rows, cols in shapes:
            x = workloads.ragged_case(rows, cols, -400, 400, seed=18, stream=rows)
            xd = to_dev(x)
            for sched in (tp.SCHED_AUTO, tp.SCHED_STREAM, tp.SCHED_CLUSTER):
                y = to_host(tp.softmax_ex(xd, workspace=ws, schedule=sched))
                assert tp.watchdog_flags(ws) == 0
                key = (rows, cols)
                if key not in refs:
                    refs[key] = y
                assert np.array_equal(y, refs[key]), (key, sched, it)


# ------------------------------------------------------------------ per-pass measurement hook

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", [(5, 16384 * 6 + 1000), (1, 1 << 20)])
def test_phase_only_reproduces_the_full_call(shape, dtype):
    # tp_phase_only (tools/pass_decomp.py): each pass alone on the stream kernel; the last pass,
    # fed the statistics of a full stream-schedule call, reproduces that call bit for bit
    x = workloads.ragged_case(*shape, -300, 300, seed=17, stream=shape[0])
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    for algo in ("two_pass", "recompute"):
        a = ALGOS[algo]
        ws = tp.new_workspace(*x.shape)
        full = to_host(tp.softmax_ex(xd, a, workspace=ws, schedule=tp.SCHED_STREAM))
        for ph in range(2 if algo == "two_pass" else 3):
            y = tp.phase_only(xd, a, ph, ws)
            assert tp.watchdog_flags(ws) == 0
        assert np.array_equal(to_host(y), full), algo
    # Reload: pass 2 alone writes exp(x - mu) into y, pass 3 alone scales it in place
    ws = tp.new_workspace(*x.shape)
    full = to_host(tp.softmax_ex(xd, tp.ALGO_RELOAD, workspace=ws, schedule=tp.SCHED_STREAM))
    tp.phase_only(xd, tp.ALGO_RELOAD, 0, ws)
    y = tp.phase_only(xd, tp.ALGO_RELOAD, 1, ws)
    tp.phase_only(xd, tp.ALGO_RELOAD, 2, ws, out=y)
    assert tp.watchdog_flags(ws) == 0
    assert np.array_equal(to_host(y), full)
    assert_parity(x, full, f"reload/{dtype}")


def test_phase_only_rejects_bad_arguments():
    xd = to_dev(workloads.ragged_case(2, 16384 * 3, seed=18))
    ws = tp.new_workspace(*xd.shape)
    for algo, ph in ((tp.ALGO_TWO_PASS, 2), (tp.ALGO_RECOMPUTE, 3), (tp.ALGO_TWO_PASS, -1), (1, 0)):
        with pytest.raises(tp.TwoPassError):
            tp.phase_only(xd, algo, ph, ws, out=torch.empty_like(xd))
    with pytest.raises(tp.TwoPassError):  # misaligned rows: the stream kernel only
        xm = to_dev(workloads.ragged_case(2, 16384 + 3, seed=18))
        tp.phase_only(xm, tp.ALGO_TWO_PASS, 0, tp.new_workspace(*xm.shape))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", [(40, 800000), (7, 16384 * 2 + 36), (20, 16384 * 100 + 8), (150, 16384 * 9),
                                       (3, 16384 * 256)])
def test_three_pass_cluster_schedule_agrees_bitwise(rows, cols, dtype):
    # the comparators on the one-cluster-per-row schedule (tp_rowcl3.cu): the stream kernel's
    # bits for every cluster size, and the oracle's tolerance
    x = workloads.ragged_case(rows, cols, -300, 300, seed=20, stream=rows + cols)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    for algo in ("recompute", "reload"):
        ref = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_STREAM))
        for cl in (0, 2, 8):
            y = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_CLUSTER, cluster_size=cl))
            assert np.array_equal(ref, y), (algo, cl, tp.last_plan())
        assert tp.watchdog_flags() == 0
        if rows * cols <= 8_000_000:
            assert_parity(x, ref, f"{algo} cluster")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_three_pass_cluster_many_rows_per_cluster(dtype):
    # a few clusters, many rows each: the bf16 kernel's software pipeline over a CTA's rows runs
    # through its four exchange buffers many times (tp_rowcl3.cu rowcl3p_kernel); fp32 the
    # sequential kernel.  Bitwise the stream kernel.
    x = workloads.ragged_case(64, 16384 * 6 + 100, -300, 300, seed=21, stream=7)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    for algo in ("recompute", "reload"):
        ref = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_STREAM))
        for cl, g in ((2, 4), (4, 4), (1, 3)):
            y = to_host(tp.softmax_ex(xd, ALGOS[algo], schedule=tp.SCHED_CLUSTER, cluster_size=cl, grid_ctas=g))
            assert np.array_equal(ref, y), (algo, cl, g, tp.last_plan())
        assert tp.watchdog_flags() == 0
        assert_parity(x, ref, f"{algo} many rows per cluster")


@pytest.mark.parametrize("cl", [1, 2])
def test_cluster_clamp_masks_with_short_shares(cl):
    # regression (found by tools/soak.py): with short shares team B of the cluster kernel could
    # trail the tree warp by two rows and read a later row's clamp masks from a per-parity shared
    # slot; masks now travel through the workspace by (row, block), and shares shorter than the
    # pass-2 pool (CL 4 here: 1 block per CTA) are not scheduled on clusters at all
    rows, cols = 93, 74316
    x = workloads.ragged_case(rows, cols, -400.0, 400.0, seed=36, stream=7)
    for r in range(0, rows, 5):  # out-of-domain elements in many rows, blocks and warps
        x[r, (r * 7919 + 62136) % cols] = 3.0e7
    xd = to_dev(x)
    ref = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    for _ in range(3):
        y = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_CLUSTER, cluster_size=cl))
        assert tp.last_plan()["kernel"] == "cluster"
        assert np.array_equal(ref, y)
    assert tp.watchdog_flags() == 0
    y4 = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_CLUSTER, cluster_size=4))
    assert tp.last_plan()["kernel"] == "stream" and np.array_equal(ref, y4)


def test_randomised_soak_short():
    # tools/soak.py for 20 s (random shapes, dtypes, algorithms, schedules, grids, out-of-domain
    # values, the partial / finish split): every output bitwise equal to the stream schedule's
    import subprocess
    import sys
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    r = subprocess.run([sys.executable, "tools/soak.py", "--minutes", "0.33", "--seed", "11", "--clamp-frac", "0.3"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


# ------------------------------------------------------------------ phase kernel (static schedule, tp_rowph.cu)

PHASE_SHAPES = [(1, 16384 * 300 + 24), (3, 16384 * 200), (1, 1 << 22), (2, 16384 * 149 + 4000), (8, 16384 * 40)]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("rows,cols", PHASE_SHAPES)
def test_phase_schedule_bitwise_and_parity(rows, cols, dtype):
    # the phase kernel (one CTA per SM, pass 1 of every block then pass 2, the block trees in a
    # tree warp) computes what every other schedule computes, bit for bit (reading G8)
    x = workloads.ragged_case(rows, cols, -2000.0, 2000.0, seed=rows + 7, stream=cols % 1000)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    y_stream = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_STREAM))
    for grid in (0, 7, 148):
        y = to_host(tp.softmax_ex(xd, schedule=tp.SCHED_PHASE, grid_ctas=grid))
        assert tp.last_plan()["kernel"] == "phase"
        assert np.array_equal(y, y_stream), grid
    assert_parity(x, y_stream, f"phase {rows}x{cols} {dtype}")


@pytest.mark.parametrize("world", [1, 2, 8])
def test_phase_schedule_partial_finish(world):
    # the chunk launches of a sharded row on the phase kernel: bitwise the one-GPU result (P9), the
    # clamp decisions of out-of-domain blocks replayed from the partial's workspace
    # row max near -2^21 with elements beyond the accuracy domain (reading G11): every 7th element
    # at -3e6 inside in-domain warps (pass 1 unclamped: they weigh 0, and must stay 0), and whole
    # blocks at -3e6 (their warps clamp to -2^21 in pass 1 and must clamp again in pass 2)
    cols = 16384 * 512
    x = workloads.ragged_case(1, cols, 0.0, 5.0, seed=71, stream=world) + np.float32(-2 ** 21 + 10)
    x[0, ::7] = -3e6
    x[0, 5 * 16384: 7 * 16384] = -3e6
    x[0, 300 * 16384 + 8192: 301 * 16384] = -3e6
    xd = to_dev(x)
    ref = to_host(tp.softmax(xd))
    from paper_2001_04438_b200 import dist as tpd
    spans = [tpd.chunk_range(cols, world, r) for r in range(world)]
    wss = [tp.new_workspace(1, b - a) for a, b in spans]
    for sched in (tp.SCHED_PHASE, tp.SCHED_STREAM):
        pairs = torch.stack([tp.partial(xd[:, a:b], workspace=w, schedule=sched)
                             for (a, b), w in zip(spans, wss)]).contiguous()
        y = torch.empty_like(xd)
        for (a, b), w in zip(spans, wss):
            tp.finish(xd[:, a:b], pairs, world, out=y[:, a:b], workspace=w, schedule=sched)
        assert np.array_equal(to_host(y), ref), sched
