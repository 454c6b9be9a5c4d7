"""Multi-GPU partitioning of the Two-Pass softmax (BASELINE.json north_star).

One process per GPU, torch.distributed for the plumbing.

  * Row sharding (config 4): rows are independent; rank k owns a contiguous block of rows
    and runs softmax_f32 on it.  No collective on the data path.
  * Chunk sharding of one long row (config 5): rank k owns the contiguous, block-aligned
    chunk k of every row.  Pass 1 gives each rank one (m, n) pair per row (8 bytes,
    Alg. 3); the pairs are exchanged with one all_gather (NCCL over
    NVLink/NVSwitch); every rank merges the `world` pairs with the same balanced tree over
    rank index inside the finish kernel (reading G8), so lambda_sum is bit-identical on all
    ranks and equal to the 1-GPU value; pass 2 then runs on the local chunk.

  * One-sided alternative: `PeerPairExchange` gives every rank a mailbox in
    its own HBM, maps the peers' mailboxes through CUDA IPC once, and exchanges the pairs with
    the library's push kernel (P2P stores over NVLink + release flags) and wait kernel
    (acquire flags): no NCCL launch per call, no host synchronisation.  Fused form: the
    partial kernel pushes each row's pair as it finishes it and releases the flag after the
    last row; the finish kernel acquires the flags itself: two launches per call in all.

The kernels are the library's (partial / finish / push / wait through the C ABI); this module
only partitions and exchanges handles.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

BLOCK_ELEMS = 16384  # canonical block size of the library (tp_common.cuh kBlockElems)


def row_range(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block of `rank` (reading G23): first rows%world ranks get one extra row."""
    base, extra = divmod(rows, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def chunk_range(cols: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous column chunk of `rank`, aligned to whole blocks (reading G23).

    When cols / world is a multiple of a power-of-two number of blocks and world is a power of
    two, every rank's pass-1 tree is a subtree of the single-GPU canonical tree and results are
    bit-identical to world = 1 (pin P9).  Otherwise chunks are still block-aligned but the
    last rank takes the remainder.
    """
    nb = -(-cols // BLOCK_ELEMS)
    per = -(-nb // world)  # blocks per rank, rounded up
    c0 = min(cols, rank * per * BLOCK_ELEMS)
    c1 = min(cols, (rank + 1) * per * BLOCK_ELEMS)
    return c0, c1


def exchange_pairs(local_pairs: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather of every rank's [rows, 2] pairs -> [world, rows, 2], rank-major (one collective)."""
    world = dist.get_world_size(group)
    rows = local_pairs.shape[0]
    out = torch.empty((world * rows, 2), dtype=local_pairs.dtype, device=local_pairs.device)
    dist.all_gather_into_tensor(out, local_pairs.contiguous(), group=group)
    return out.view(world, rows, 2)


def gather_handles(local: bytes, group=None) -> list[bytes]:
    """Every rank's IPC handle, rank-ordered (host plumbing; gloo or NCCL object collective)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local, group=group)
    return out


class PeerPairExchange:
    """One-sided NVLink exchange of [rows, 2] pairs (include/twopass.h tp_pairs_push / wait).

    `mailboxes` is normally None (one process per GPU: the mailboxes are shared with CUDA IPC
    over `group`); a list of world mailbox tensors on one device runs world emulated ranks in
    one process (tests: every push precedes every wait, so no kernel waits on another).
    """

    def __init__(self, rows: int, device, group=None, rank: int | None = None, world: int | None = None,
                 mailboxes: list[torch.Tensor] | None = None, timeout_s: float = 5.0):
        import ctypes

        import paper_2001_04438_b200 as tp
        self.tp, self.rows = tp, rows
        self.world = world if world is not None else dist.get_world_size(group)
        self.rank = rank if rank is not None else dist.get_rank(group)
        L = tp.lib()
        nbytes = int(L.tp_mailbox_bytes(self.world, rows))
        if nbytes == 0:
            raise ValueError("world must be 1..56")
        self._opened = []
        if mailboxes is not None:
            self.mailbox = mailboxes[self.rank]
            ptrs = [m.data_ptr() for m in mailboxes]
        else:
            self.mailbox = torch.zeros(nbytes, dtype=torch.uint8, device=device)
            h, off = ctypes.create_string_buffer(64), ctypes.c_uint64()
            tp._check(L.tp_ipc_get_handle(self.mailbox.data_ptr(), h, ctypes.byref(off)), "tp_ipc_get_handle")
            mine = h.raw + int(off.value).to_bytes(8, "little")
            handles = gather_handles(mine, group) if self.world > 1 else [mine]
            ptrs = []
            for r, hr in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self.mailbox.data_ptr())
                    continue
                p = ctypes.c_void_p()
                tp._check(L.tp_ipc_open(hr[:64], int.from_bytes(hr[64:72], "little"), ctypes.byref(p)),
                          "tp_ipc_open")
                self._opened.append(p.value)
                ptrs.append(p.value)
        self.peer_ptrs = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self.epoch = 0
        self.timeout_ns = int(timeout_s * 1e9)

    def _next_epoch(self) -> int:
        """1, 2, ..., 2^32 - 2, 1, ...: never 0 (the zero-filled state), parity alternating."""
        return self.epoch % 0xFFFFFFFE + 1

    def push(self, local_pairs: torch.Tensor, epoch: int) -> None:
        tp = self.tp
        tp._check(tp.lib().tp_pairs_push(local_pairs.data_ptr(), self.rows, self.peer_ptrs.data_ptr(), self.rank,
                                         self.world, epoch, tp._stream()), "tp_pairs_push")

    def wait(self, epoch: int) -> torch.Tensor:
        """The [world, rows, 2] pairs of this epoch in the local mailbox (stream-ordered)."""
        tp = self.tp
        tp._check(tp.lib().tp_pairs_wait(self.mailbox.data_ptr(), self.world, epoch, self.timeout_ns,
                                         tp._stream()), "tp_pairs_wait")
        return self.pairs(epoch)

    def pairs(self, epoch: int | None = None) -> torch.Tensor:
        """The pairs half of `epoch` (default: the last epoch used) of the local mailbox."""
        e = self.epoch if epoch is None else epoch
        off = int(self.tp.lib().tp_mailbox_pairs_offset(self.world, self.rows, e))
        return self.mailbox[off:off + 8 * self.world * self.rows].view(torch.float32).view(self.world, self.rows, 2)

    def error(self) -> int:
        """Bit r: the last waits timed out on rank r (reads device memory: synchronises)."""
        return int(self.mailbox[512:516].view(torch.int32).item())

    def exchange(self, local_pairs: torch.Tensor) -> torch.Tensor:
        self.epoch = self._next_epoch()
        self.push(local_pairs, self.epoch)
        return self.wait(self.epoch)

    # fused path: pass 1 pushes its pairs from inside the partial kernel and the finish kernel
    # awaits them itself (softmax_partial_push_ex / softmax_finish_mailbox_ex): two launches

    def push_partial(self, x_chunk: torch.Tensor, workspace: torch.Tensor | None = None) -> int:
        """Pass 1 of this rank's chunk with the in-kernel push; returns the epoch to finish with."""
        self.epoch = self._next_epoch()
        if x_chunk.shape[-1] == 0:  # an empty trailing chunk contributes the identity (0, -inf)
            ident = torch.tensor([[0.0, float("-inf")]] * self.rows, dtype=torch.float32, device=x_chunk.device)
            self.push(ident, self.epoch)
        else:
            self.tp.partial_push(x_chunk, self.peer_ptrs, self.rank, self.world, self.epoch, workspace=workspace)
        return self.epoch

    def finish(self, x_chunk: torch.Tensor, epoch: int, out: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None) -> torch.Tensor:
        """Await `epoch` in the local mailbox inside the finish kernel, merge, pass 2 (`workspace`:
        the one push_partial used)."""
        if x_chunk.shape[-1] == 0:
            self.wait(epoch)
            return torch.empty(x_chunk.shape, dtype=torch.float32, device=x_chunk.device) if out is None else out
        return self.tp.finish_mailbox(x_chunk, self.mailbox, self.world, epoch, self.timeout_ns, out=out,
                                      workspace=workspace)

    def close(self) -> None:
        for p in self._opened:
            self.tp.lib().tp_ipc_close(p)
        self._opened = []


def chunk_sharded_softmax(x_chunk: torch.Tensor, out: torch.Tensor | None = None, group=None,
                          workspace: torch.Tensor | None = None,
                          exchange: "PeerPairExchange | None" = None, fused: bool = False) -> torch.Tensor:
    """Softmax of rows sharded by column chunk: partial -> exchange 8 B/row/rank -> finish.

    The exchange is one NCCL all_gather, or the one-sided NVLink mailboxes when `exchange` is
    given: push / wait kernels between partial and finish, or (fused) pushed by the partial
    kernel itself and awaited by the finish kernel itself."""
    import paper_2001_04438_b200 as tp
    if exchange is not None and fused:
        return exchange.finish(x_chunk, exchange.push_partial(x_chunk, workspace), out=out, workspace=workspace)
    rows = x_chunk.shape[0]
    if x_chunk.shape[-1] == 0:  # an empty trailing chunk contributes the identity (0, -inf)
        pairs = torch.tensor([[0.0, float("-inf")]] * rows, dtype=torch.float32, device=x_chunk.device)
        if exchange is not None:
            exchange.exchange(pairs)
        else:
            exchange_pairs(pairs, group)
        return torch.empty(x_chunk.shape, dtype=torch.float32, device=x_chunk.device) if out is None else out
    pairs = tp.partial(x_chunk, workspace=workspace)
    allp = exchange.exchange(pairs) if exchange is not None else exchange_pairs(pairs, group)
    return tp.finish(x_chunk, allp, allp.shape[0], out=out, workspace=workspace)


def gather_rows(v: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather of every rank's [rows] values -> [world, rows], rank-major (one collective)."""
    world = dist.get_world_size(group)
    out = torch.empty((world * v.numel(),), dtype=v.dtype, device=v.device)
    dist.all_gather_into_tensor(out, v.contiguous(), group=group)
    return out.view(world, v.numel())


def chunk_sharded_softmax3(x_chunk: torch.Tensor, algo: int, out: torch.Tensor | None = None, group=None,
                           workspace: torch.Tensor | None = None) -> torch.Tensor:
    """The Three-Pass comparators (Alg. 1 Recompute / Alg. 2 Reload) on rows
    sharded by column chunk: TWO exchanges per call, where the Two-Pass needs one:
    max partial -> all_gather -> sum partial (Reload writes exp(x - mu)) -> all_gather -> finish.
    Gathering (not all-reducing) keeps the merge in the kernels' canonical rank-order tree, so
    the result is bitwise that of one GPU for power-of-two worlds."""
    import paper_2001_04438_b200 as tp
    rows = x_chunk.shape[0]
    if x_chunk.shape[-1] == 0:  # an empty trailing chunk: max -inf, sum 0
        gather_rows(torch.full((rows,), float("-inf"), device=x_chunk.device), group)
        gather_rows(torch.zeros(rows, device=x_chunk.device), group)
        return torch.empty(x_chunk.shape, dtype=torch.float32, device=x_chunk.device) if out is None else out
    y = torch.empty(x_chunk.shape, dtype=torch.float32, device=x_chunk.device) if out is None else out
    maxes = gather_rows(tp.softmax3_max_partial(x_chunk, workspace=workspace), group)
    sums = gather_rows(tp.softmax3_sum_partial(x_chunk, algo, maxes, out=y, workspace=workspace), group)
    return tp.softmax3_finish(x_chunk, algo, maxes, sums, out=y, workspace=workspace)


def row_sharded_softmax(x_rows: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Softmax of a rank's own rows: no communication."""
    import paper_2001_04438_b200 as tp
    return tp.softmax(x_rows, out=out)


class HostChunkPipeline:
    """End-to-end chunk-sharded softmax of one row from and to HOST (pinned) buffers of this
    rank's chunk (the multi-GPU counterpart of softmax_f32_host).

    The chunk is cut into `nsub` equal block-aligned sub-chunks (a power of two).  The H2D copy of
    sub-chunk k (copy stream) overlaps pass 1 of sub-chunk k - 1 (compute stream, one
    softmax_partial per sub-chunk, each with its own workspace); the world x nsub pairs are
    gathered in one all_gather (rank-major, then sub-chunk order: the canonical tree over them is
    the one-GPU tree, reading G8); the finish of sub-chunk k (merging world x nsub pairs) overlaps
    the D2H copy of sub-chunk k - 1.  Device buffers, streams and workspaces are kept between
    calls.  Every arithmetic step runs in the library's kernels.
    """

    def __init__(self, cols: int, device, dtype=torch.float32, nsub: int = 8, group=None):
        import paper_2001_04438_b200 as tp
        self.tp, self.group, self.device = tp, group, torch.device(device)
        while nsub > 1 and cols % (BLOCK_ELEMS * nsub):  # equal block-aligned sub-chunks only
            nsub //= 2
        self.nsub, self.cols = nsub, cols
        self.sub = cols // nsub if nsub > 1 else cols
        self.dx = torch.empty((1, cols), dtype=dtype, device=self.device)
        self.dy = torch.empty((1, cols), dtype=torch.float32, device=self.device)
        self.ws = [tp.new_workspace(1, self.sub, self.device) for _ in range(nsub)]
        self.pairs = torch.empty((nsub, 1, 2), dtype=torch.float32, device=self.device)
        self.copy = torch.cuda.Stream(self.device)
        self.comp = torch.cuda.Stream(self.device)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def _span(self, k):
        return slice(k * self.sub, self.cols if k == self.nsub - 1 else (k + 1) * self.sub)

    def run(self, hx: torch.Tensor, hy: torch.Tensor) -> torch.Tensor:
        tp, n = self.tp, self.nsub
        assert hx.shape == (1, self.cols) and hy.shape == (1, self.cols)
        cur = torch.cuda.current_stream(self.device)
        self.copy.wait_stream(cur)
        self.comp.wait_stream(cur)
        h2d = []
        for k in range(n):  # H2D of k || pass 1 of k - 1
            sp = self._span(k)
            with torch.cuda.stream(self.copy):
                self.dx[:, sp].copy_(hx[:, sp], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy)
                h2d.append(ev)
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(ev)
                tp.partial(self.dx[:, sp], out=self.pairs[k], workspace=self.ws[k])
        with torch.cuda.stream(self.comp):
            if self.world > 1:
                allp = torch.empty((self.world * n, 1, 2), dtype=torch.float32, device=self.device)
                dist.all_gather_into_tensor(allp.view(-1), self.pairs.view(-1), group=self.group)
            else:
                allp = self.pairs
            for k in range(n):  # finish of k || D2H of k - 1
                sp = self._span(k)
                tp.finish(self.dx[:, sp], allp, self.world * n, out=self.dy[:, sp], workspace=self.ws[k])
                ev = torch.cuda.Event()
                ev.record(self.comp)
                with torch.cuda.stream(self.copy):
                    self.copy.wait_event(ev)
                    hy[:, sp].copy_(self.dy[:, sp], non_blocking=True)
        self.copy.synchronize()
        return hy
