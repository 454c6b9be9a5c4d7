"""Sharded Three-Pass comparators and the NCCL path on the GPU (BASELINE.json
metric "vs three-pass, at 1/2/4/8 B200").

One GPU here: W ranks are emulated on one device for the kernels (every partial before every
merge, so no kernel waits on another), the real collective runs as a world-1 NCCL group on
cuda:0, and a torchrun world-2 run is exercised when two GPUs are visible.
"""
import os
import socket
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
ALGO3 = {"recompute": tp.ALGO_RECOMPUTE, "reload": tp.ALGO_RELOAD}


def _chunks(xd, world):
    return [xd[:, slice(*tpd.chunk_range(xd.shape[1], world, r))].contiguous() for r in range(world)]


def _sharded3(xd, algo, world, per_rank_ws=True):
    """Alg. 1 / 2 over W emulated ranks: max partials -> gathered -> sum partials -> gathered ->
    finishes (what dist.chunk_sharded_softmax3 does with all_gather between the steps)."""
    ch = _chunks(xd, world)
    live = [c for c in ch if c.shape[1]]
    wss = [tp.new_workspace(c.shape[0], c.shape[1]) if per_rank_ws else None for c in live]
    rows = xd.shape[0]
    ninf = torch.full((rows,), float("-inf"), device="cuda")
    maxes = torch.stack([tp.softmax3_max_partial(c, workspace=w) for c, w in zip(live, wss)] +
                        [ninf] * (world - len(live))).contiguous()
    ys = [torch.empty(c.shape, dtype=torch.float32, device="cuda") for c in live]
    sums = torch.stack([tp.softmax3_sum_partial(c, algo, maxes, out=y, workspace=w) for c, y, w in zip(live, ys, wss)]
                       + [torch.zeros(rows, device="cuda")] * (world - len(live))).contiguous()
    outs = [tp.softmax3_finish(c, algo, maxes, sums, out=y, workspace=w) for c, y, w in zip(live, ys, wss)]
    return np.concatenate([to_host(o) for o in outs], axis=1)


@pytest.mark.parametrize("algo", list(ALGO3))
@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("rows,cols,dtype", [(1, 16384 * 64, "f32"), (3, 16384 * 8 + 96, "f32"),
                                             (2, 16384 * 16, "bf16"), (1, 16384 * 8 + 1, "f32")])
def test_sharded_three_pass_matches_one_gpu(algo, world, rows, cols, dtype):
    x = workloads.ragged_case(rows, cols, -1000, 1000, seed=41, stream=world)
    if dtype == "bf16":
        x = workloads.to_bf16(x)
    xd = to_dev(x)
    ref = to_host(tp.softmax_ex(xd, ALGO3[algo], schedule=tp.SCHED_STREAM))
    y = _sharded3(xd, ALGO3[algo], world)
    assert_parity(x, y, f"sharded {algo} W={world}")
    if cols % (16384 * world) == 0:
        assert np.array_equal(y, ref)  # canonical trees: bitwise the one-GPU comparator (P9)


def test_sharded_three_pass_world1_is_the_plain_comparator():
    x = workloads.generate("c3")
    xd = to_dev(x)
    for algo in ALGO3.values():
        ref = to_host(tp.softmax_ex(xd, algo))
        assert np.array_equal(_sharded3(xd, algo, 1), ref)


def test_sharded_three_pass_rejects_bad_arguments():
    xd = to_dev(workloads.ragged_case(2, 16384, seed=3))
    L = tp.lib()
    st = tp._stream()
    m = torch.empty(2, device="cuda")
    assert L.softmax3_max_partial_ex(tp.IN_F32, xd.data_ptr(), 2, 16384, None, None, 0, st) == tp.TP_EINVAL
    assert L.softmax3_sum_partial_ex(tp.ALGO_TWO_PASS, tp.IN_F32, xd.data_ptr(), None, 2, 16384, m.data_ptr(), 1,
                                     m.data_ptr(), None, 0, st) == tp.TP_EINVAL
    assert L.softmax3_sum_partial_ex(tp.ALGO_RELOAD, tp.IN_F32, xd.data_ptr(), None, 2, 16384, m.data_ptr(), 1,
                                     m.data_ptr(), None, 0, st) == tp.TP_EINVAL   # Reload writes y
    assert L.softmax3_finish_ex(tp.ALGO_RECOMPUTE, tp.IN_F32, xd.data_ptr(), None, 2, 16384, m.data_ptr(),
                                m.data_ptr(), 1, None, 0, st) == tp.TP_EINVAL


# ------------------------------------------------------------------ the real collective (NCCL)

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world1_chunk_sharded_paths():
    # dist.chunk_sharded_softmax (partial -> all_gather_into_tensor over NCCL -> finish) and
    # dist.chunk_sharded_softmax3 (two all_gathers) in a real NCCL process group of one rank on
    # cuda:0: bitwise the plain calls
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = workloads.generate("c3")
        xd = to_dev(x)
        ws = tp.new_workspace(1, x.shape[1])
        y = tpd.chunk_sharded_softmax(xd, workspace=ws)
        assert torch.equal(y, tp.softmax(xd))
        for algo in ALGO3.values():
            y3 = tpd.chunk_sharded_softmax3(xd, algo, workspace=ws)
            assert torch.equal(y3, tp.softmax_ex(xd, algo))
        assert_parity(x, to_host(y), "nccl world 1")
    finally:
        dist.destroy_process_group()


TORCHRUN_CHILD = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import paper_2001_04438_b200 as tp, workloads
from paper_2001_04438_b200 import dist as tpd
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
x = torch.from_numpy(workloads.generate("c3")).cuda()
c0, c1 = tpd.chunk_range(x.shape[1], world, rank)
xc = x[:, c0:c1].contiguous()
ref = tp.softmax(x)[:, c0:c1]
assert torch.equal(tpd.chunk_sharded_softmax(xc), ref)
for algo in (tp.ALGO_RECOMPUTE, tp.ALGO_RELOAD):
    assert torch.equal(tpd.chunk_sharded_softmax3(xc, algo), tp.softmax_ex(x, algo)[:, c0:c1])
ex = tpd.PeerPairExchange(1, "cuda")
for _ in range(3):
    assert torch.equal(tpd.chunk_sharded_softmax(xc, exchange=ex), ref)
    assert torch.equal(tpd.chunk_sharded_softmax(xc, exchange=ex, fused=True), ref)
dist.barrier()
ex.close()
dist.destroy_process_group()
print("rank", rank, "ok")
"""


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (one process per GPU)")
def test_torchrun_world2_chunk_sharded(tmp_path):
    script = tmp_path / "child.py"
    script.write_text(TORCHRUN_CHILD)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(script), ROOT],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
