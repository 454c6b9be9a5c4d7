"""Multi-GPU host logic on CPU (-m "not gpu"): partitioning and the (m, n) pair exchange
with world-size-2 gloo process groups (the kernels themselves run on GPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2001_04438_b200 import dist as tpd


@pytest.mark.parametrize("rows,world", [(256, 1), (256, 2), (256, 8), (7, 4), (3, 8)])
def test_row_range_partitions_rows(rows, world):
    spans = [tpd.row_range(rows, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == rows
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0 and a0 <= a1
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("cols,world", [(1 << 31, 1), (1 << 31, 2), (1 << 31, 8), (800000, 4), (1 << 26, 8),
                                        (16384 * 5 + 3, 4)])
def test_chunk_range_is_block_aligned_and_covers(cols, world):
    spans = [tpd.chunk_range(cols, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == cols
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    for a0, a1 in spans:
        assert a0 % tpd.BLOCK_ELEMS == 0 or a0 == a1 == cols   # empty trailing chunks allowed
    if cols % (world * tpd.BLOCK_ELEMS) == 0:
        nblk = {(a1 - a0) // tpd.BLOCK_ELEMS for a0, a1 in spans}
        assert len(nblk) == 1                      # equal chunks
        n = nblk.pop()
        if (cols // tpd.BLOCK_ELEMS) & ((cols // tpd.BLOCK_ELEMS) - 1) == 0:
            assert n & (n - 1) == 0                # power-of-two runs of blocks: subtrees of G8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = 3
    local = torch.tensor([[rank + 1.0, 10.0 * rank + r] for r in range(rows)], dtype=torch.float32)
    allp = tpd.exchange_pairs(local)
    # the layout the finish kernel reads: [world, rows, 2], rank-major
    out_q.put((rank, allp.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_pair_exchange_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=60) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [[[w + 1.0, 10.0 * w + r] for r in range(3)] for w in range(world)]
    assert res[0] == want and res[1] == want           # every rank holds every pair, rank-major


def _handles_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2001_04438_b200 import dist as tpd
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q.put((rank, tpd.gather_handles(bytes([rank]) * 64)))
    finally:
        dist.destroy_process_group()


def test_ipc_handles_gathered_rank_ordered():
    # NEXT-4 plumbing: every rank sees every rank's 64-byte mailbox handle, in rank order
    import multiprocessing as mp
    import socket
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ps = [ctx.Process(target=_handles_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert res[r] == [bytes([0]) * 64, bytes([1]) * 64]


# ---- the sharded Three-Pass orchestration (dist.chunk_sharded_softmax3) with gloo: the kernels
# are replaced by plain CPU stand-ins of the same per-chunk contract (the host logic under test is
# the sequence max partial -> gather -> sum partial -> gather -> finish and the rank order)

def _fake_tp():
    import types
    import paper_2001_04438_b200 as real
    f = types.SimpleNamespace(ALGO_RECOMPUTE=real.ALGO_RECOMPUTE, ALGO_RELOAD=real.ALGO_RELOAD)
    f.softmax3_max_partial = lambda x, workspace=None: x.double().amax(dim=1).float()

    def sum_partial(x, algo, maxes, out=None, workspace=None):
        mu = maxes.amax(dim=0).double()
        e = torch.exp(x.double() - mu[:, None])
        if algo == real.ALGO_RELOAD:
            out.copy_(e.float())
        return e.sum(dim=1).float()

    def finish(x, algo, maxes, sums, out=None, workspace=None):
        mu = maxes.amax(dim=0).double()
        sigma = sums.double().sum(dim=0)
        e = torch.exp(x.double() - mu[:, None]) if algo == real.ALGO_RECOMPUTE else out.double()
        out.copy_((e / sigma[:, None]).float())
        return out
    f.softmax3_sum_partial, f.softmax3_finish = sum_partial, finish
    return f


def _sharded3_worker(rank, world, port, q):
    import sys
    import paper_2001_04438_b200 as real
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        sys.modules["paper_2001_04438_b200"] = _fake_tp()
        torch.manual_seed(0)
        x = torch.randn(3, 40, dtype=torch.float64).float() * 30
        c0, c1 = rank * 20, rank * 20 + 20
        outs = {}
        for algo in (real.ALGO_RECOMPUTE, real.ALGO_RELOAD):
            outs[algo] = tpd.chunk_sharded_softmax3(x[:, c0:c1].contiguous(), algo).tolist()
        want = torch.softmax(x.double(), dim=1)[:, c0:c1]
        q.put((rank, [float((torch.tensor(v, dtype=torch.float64) - want).abs().max()) for v in outs.values()]))
    finally:
        sys.modules["paper_2001_04438_b200"] = real
        dist.destroy_process_group()


def test_chunk_sharded_three_pass_orchestration_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_sharded3_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert max(res[r]) < 1e-6, res[r]
