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

The kernels are the library's (partial / finish through the C ABI); this module only
partitions and exchanges.
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


def chunk_sharded_softmax(x_chunk: torch.Tensor, out: torch.Tensor | None = None, group=None,
                          workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Softmax of rows sharded by column chunk: partial -> all_gather(8 B/row/rank) -> finish."""
    import paper_2001_04438_b200 as tp
    rows = x_chunk.shape[0]
    if x_chunk.shape[-1] == 0:  # an empty trailing chunk contributes the identity (0, -inf)
        pairs = torch.tensor([[0.0, float("-inf")]] * rows, dtype=torch.float32, device=x_chunk.device)
        exchange_pairs(pairs, group)
        return torch.empty(x_chunk.shape, dtype=torch.float32, device=x_chunk.device) if out is None else out
    pairs = tp.partial(x_chunk, workspace=workspace)
    allp = exchange_pairs(pairs, group)
    return tp.finish(x_chunk, allp, allp.shape[0], out=out)


def row_sharded_softmax(x_rows: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Softmax of a rank's own rows: no communication."""
    import paper_2001_04438_b200 as tp
    return tp.softmax(x_rows, out=out)
