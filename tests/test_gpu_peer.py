"""One-sided NVLink pair exchange (include/twopass.h tp_pairs_push / wait).

One GPU here: W ranks are emulated on one device (every push precedes every wait, so no kernel
waits on another kernel), and the CUDA IPC mapping is exercised with a second process that
pushes into this process's mailbox and exits before this process waits.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import workloads
from gpu_helpers import assert_parity, to_dev, to_host

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2001_04438_b200")
from paper_2001_04438_b200 import dist as tpd  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _chunks(x, world):
    return [x[:, slice(*tpd.chunk_range(x.shape[1], world, r))] for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("rows,cols", [(1, 16384 * 64), (3, 16384 * 8 + 96)])
def test_mailbox_exchange_matches_allgather_and_one_gpu(world, rows, cols):
    x = workloads.ragged_case(rows, cols, -1000, 1000, seed=21, stream=world)
    xd = to_dev(x)
    ref = to_host(tp.softmax(xd))
    nbytes = tp.lib().tp_mailbox_bytes(world, rows)
    boxes = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    ex = [tpd.PeerPairExchange(rows, "cuda", rank=r, world=world, mailboxes=boxes) for r in range(world)]
    chunks = [c.contiguous() for c in _chunks(xd, world)]
    ident = torch.tensor([[0.0, float("-inf")]] * rows, dtype=torch.float32, device="cuda")
    for epoch in (1, 2):  # reuse without resetting the mailboxes
        # an empty trailing chunk contributes the identity pair (dist.chunk_sharded_softmax)
        parts = [tp.partial(c) if c.shape[1] else ident for c in chunks]
        for r in range(world):
            ex[r].push(parts[r], epoch)
        outs = []
        for r in range(world):
            allp = ex[r].wait(epoch)
            assert torch.equal(allp, torch.stack(parts))          # same bytes as an all_gather
            if chunks[r].shape[1]:
                outs.append(to_host(tp.finish(chunks[r], allp, world)))
        y = np.concatenate(outs, axis=1)
        assert all(e.error() == 0 for e in ex)
        # power-of-two worlds over power-of-two block runs: bit-identical to one GPU (pin P9)
        if cols % (16384 * world) == 0:
            assert np.array_equal(y, ref)
        else:
            assert_parity(x, y, f"mailbox W={world}")


def test_wait_times_out_instead_of_hanging():
    ex = tpd.PeerPairExchange(2, "cuda", rank=0, world=2,
                              mailboxes=[torch.zeros(tp.lib().tp_mailbox_bytes(2, 2), dtype=torch.uint8,
                                                     device="cuda") for _ in range(2)], timeout_s=0.002)
    ex.push(torch.zeros((2, 2), dtype=torch.float32, device="cuda"), 7)
    ex.wait(7)                        # rank 1 never pushes
    torch.cuda.synchronize()
    assert ex.error() == 0b10


CHILD = r"""
import sys, ctypes, torch
sys.path.insert(0, sys.argv[1])
import paper_2001_04438_b200 as tp, workloads
from paper_2001_04438_b200 import dist as tpd
handle = bytes.fromhex(sys.argv[2])
offset = int(sys.argv[3])
x = torch.from_numpy(workloads.ragged_case(2, 16384 * 4, -50, 50, seed=5, stream=5)).cuda()
c1 = x[:, slice(*tpd.chunk_range(x.shape[1], 2, 1))].contiguous()
p = ctypes.c_void_p()
assert tp.lib().tp_ipc_open(handle, offset, ctypes.byref(p)) == 0
mine = torch.zeros(tp.lib().tp_mailbox_bytes(2, 2), dtype=torch.uint8, device="cuda")
peers = torch.tensor([p.value, mine.data_ptr()], dtype=torch.int64, device="cuda")
pairs = tp.partial(c1)
assert tp.lib().tp_pairs_push(pairs.data_ptr(), 2, peers.data_ptr(), 1, 2, 3, tp._stream()) == 0
torch.cuda.synchronize()
assert tp.lib().tp_ipc_close(p) == 0
print("pushed")
"""


def test_ipc_mailbox_written_by_another_process():
    import ctypes
    x = workloads.ragged_case(2, 16384 * 4, -50, 50, seed=5, stream=5)
    xd = to_dev(x)
    box = torch.zeros(tp.lib().tp_mailbox_bytes(2, 2), dtype=torch.uint8, device="cuda")
    h, off = ctypes.create_string_buffer(64), ctypes.c_uint64()
    assert tp.lib().tp_ipc_get_handle(box.data_ptr(), h, ctypes.byref(off)) == 0
    torch.cuda.synchronize()
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, h.raw.hex(), str(off.value)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "pushed" in r.stdout, r.stderr[-2000:]
    ex = tpd.PeerPairExchange(2, "cuda", rank=0, world=2, mailboxes=[box, torch.zeros_like(box)])
    c0 = xd[:, slice(*tpd.chunk_range(x.shape[1], 2, 0))].contiguous()
    ex.push(tp.partial(c0), 3)
    allp = ex.wait(3)
    torch.cuda.synchronize()
    assert ex.error() == 0
    c1 = xd[:, slice(*tpd.chunk_range(x.shape[1], 2, 1))].contiguous()
    assert torch.equal(allp[1], tp.partial(c1))                 # rank 1's pairs arrived through IPC
    y = np.concatenate([to_host(tp.finish(c0, allp, 2)), to_host(tp.finish(c1, allp, 2))], axis=1)
    assert np.array_equal(y, to_host(tp.softmax(xd)))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("rows,cols,dtype", [(1, 16384 * 64, "f32"), (3, 16384 * 8 + 96, "f32"),
                                             (2, 16384 * 16, "bf16")])
def test_fused_push_and_in_kernel_wait(world, rows, cols, dtype):
    # softmax_partial_push_ex / softmax_finish_mailbox_ex: the partial kernel pushes its pairs and
    # releases the flag itself, the finish kernel awaits the flags itself; emulated ranks, every
    # partial before every finish (no kernel waits on another)
    x = workloads.ragged_case(rows, cols, -1000, 1000, seed=22, stream=world)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ref = to_host(tp.softmax(xd))
    nbytes = tp.lib().tp_mailbox_bytes(world, rows)
    boxes = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    ex = [tpd.PeerPairExchange(rows, "cuda", rank=r, world=world, mailboxes=boxes) for r in range(world)]
    chunks = [c.contiguous() for c in _chunks(xd, world)]
    wss = [tp.new_workspace(rows, max(c.shape[1], 1)) for c in chunks]  # one per emulated rank
    for _ in range(3):  # epochs 1, 2, 3 on the same mailboxes
        epochs = [ex[r].push_partial(chunks[r], wss[r]) for r in range(world)]
        outs = [to_host(ex[r].finish(chunks[r], epochs[r], workspace=wss[r])) for r in range(world)
                if chunks[r].shape[1]]
        assert tp.watchdog_flags() == 0 and all(e.error() == 0 for e in ex)
        # the mailbox holds exactly the pairs the unfused partial computes
        parts = torch.stack([tp.partial(c) if c.shape[1] else
                             torch.tensor([[0.0, float("-inf")]] * rows, device="cuda") for c in chunks])
        assert all(torch.equal(e.pairs(), parts) for e in ex)
        y = np.concatenate(outs, axis=1)
        if cols % (16384 * world) == 0:
            assert np.array_equal(y, ref)
        else:
            assert_parity(x, y, f"fused W={world}")


def test_fused_finish_times_out_instead_of_hanging():
    rows, world = 2, 2
    boxes = [torch.zeros(tp.lib().tp_mailbox_bytes(world, rows), dtype=torch.uint8, device="cuda")
             for _ in range(world)]
    ex = tpd.PeerPairExchange(rows, "cuda", rank=0, world=world, mailboxes=boxes, timeout_s=0.002)
    xd = to_dev(workloads.ragged_case(rows, 16384 * 2, seed=23))
    ep = ex.push_partial(xd)
    ex.finish(xd, ep)                 # rank 1 never pushes
    torch.cuda.synchronize()
    assert ex.error() == 0b10
    assert tp.watchdog_flags() & 1    # reported (and cleared) by the watchdog
    y = tp.softmax(xd)                # the workspace is usable again afterwards
    assert_parity(to_host(xd), to_host(y), "after timeout")


@pytest.mark.parametrize("fused", [False, True])
def test_mailbox_reuse_with_a_rank_one_epoch_ahead(fused):
    # Rank A finishes epoch 1 and pushes epoch 2 (new data) before rank B's finish of epoch 1 has
    # read the pairs: the epoch-parity halves keep B's epoch-1 pairs intact (a single-buffered
    # mailbox fails here: B's flag wait sees epoch 2, or B reads A's epoch-2 pair).  Emulated
    # ranks, one stream, every wait after the pushes it needs (no kernel waits on another).
    world, rows, cols = 2, 3, 16384 * 8
    xs = [workloads.ragged_case(rows, cols, -300, 300, seed=31 + e, stream=9) for e in (1, 2)]
    xds = [to_dev(x) for x in xs]
    refs = [to_host(tp.softmax(xd)) for xd in xds]
    ch = [[c.contiguous() for c in _chunks(xd, world)] for xd in xds]
    nbytes = tp.lib().tp_mailbox_bytes(world, rows)
    boxes = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    ex = [tpd.PeerPairExchange(rows, "cuda", rank=r, world=world, mailboxes=boxes) for r in range(world)]
    wss = [tp.new_workspace(rows, cols // world) for _ in range(world)]
    if fused:
        e1 = [ex[r].push_partial(ch[0][r], wss[r]) for r in range(world)]
        ya1 = ex[0].finish(ch[0][0], e1[0], workspace=wss[0])
        e2a = ex[0].push_partial(ch[1][0], wss[0])              # A one epoch ahead
        yb1 = ex[1].finish(ch[0][1], e1[1], workspace=wss[1])  # B still on epoch 1
        e2b = ex[1].push_partial(ch[1][1], wss[1])
        ya2 = ex[0].finish(ch[1][0], e2a, workspace=wss[0])
        yb2 = ex[1].finish(ch[1][1], e2b, workspace=wss[1])
    else:
        def part(e, r):
            return tp.partial(ch[e][r], workspace=wss[r])
        p1 = [part(0, r) for r in range(world)]
        for r in range(world):
            ex[r].push(p1[r], 1)
        ya1 = tp.finish(ch[0][0], ex[0].wait(1), world, workspace=wss[0]).clone()
        ex[0].push(part(1, 0), 2)                               # A one epoch ahead
        yb1 = tp.finish(ch[0][1], ex[1].wait(1), world, workspace=wss[1]).clone()
        ex[1].push(part(1, 1), 2)
        ya2 = tp.finish(ch[1][0], ex[0].wait(2), world, workspace=wss[0])
        yb2 = tp.finish(ch[1][1], ex[1].wait(2), world, workspace=wss[1])
    torch.cuda.synchronize()
    assert all(e.error() == 0 for e in ex) and tp.watchdog_flags() == 0
    assert np.array_equal(np.concatenate([to_host(ya1), to_host(yb1)], axis=1), refs[0])
    assert np.array_equal(np.concatenate([to_host(ya2), to_host(yb2)], axis=1), refs[1])


def test_watchdog_abort_is_reported_by_the_next_call():
    # a launch that gives up a wait (here: the fused finish whose peer never pushes) makes the
    # NEXT call on the device fail with TP_EWATCHDOG; the call after that runs normally
    rows, world = 2, 2
    boxes = [torch.zeros(tp.lib().tp_mailbox_bytes(world, rows), dtype=torch.uint8, device="cuda")
             for _ in range(world)]
    ex = tpd.PeerPairExchange(rows, "cuda", rank=0, world=world, mailboxes=boxes, timeout_s=0.002)
    x = workloads.ragged_case(rows, 16384 * 2, seed=24)
    xd = to_dev(x)
    ex.finish(xd, ex.push_partial(xd))  # rank 1 never pushes: the in-kernel wait gives up
    torch.cuda.synchronize()
    with pytest.raises(tp.TwoPassError, match="watchdog"):
        tp.softmax(xd)
    y = tp.softmax(xd)                  # state was reset by the reporting call
    assert_parity(x, to_host(y), "after a reported abort")
    assert tp.watchdog_flags() == 0
