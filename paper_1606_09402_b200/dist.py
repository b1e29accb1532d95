"""Row sharding of A over the GPUs of one box (one process per GPU).

A = [A_1; ...; A_G] by rows. G = A*Omega, Y, Q live row-sharded; Omega, B^T and every
n-side block are replicated (each rank generates the identical Omega from the seed
and performs the identical replicated arithmetic). The device engine allreduces
(NCCL over NVLink/NVSwitch) exactly:
  * the n x w result of every A^T pass (H = A^T G, B_i^T = A^T Q_i, power A^T Y),
  * the b x b / k x b Grams over rows (Y^T Y, Q^T Y, Q^T Q_i),
  * the scalar ||A||_F^2.
This module holds the host side: shard planning (dense: even, aligned row blocks;
CSR: balanced by nnz + rows), slicing, and the NCCL bootstrap through an existing
torch.distributed process group.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def plan_dense_rows(m: int, world: int, align: int = 32) -> List[Tuple[int, int]]:
    """Even row blocks with interior boundaries on multiples of `align` (16-byte aligned
    row offsets for the DMMA tile loads). Returns [(row0, rows)] per rank."""
    if world < 1:
        raise ValueError("world must be >= 1")
    bounds = [0]
    for g in range(1, world):
        b = int(round(m * g / world / align)) * align
        bounds.append(min(max(b, bounds[-1]), m))
    bounds.append(m)
    return [(bounds[g], bounds[g + 1] - bounds[g]) for g in range(world)]


def plan_csr_rows(row_ptr, world: int, row_weight: float = 1.0) -> List[Tuple[int, int]]:
    """Contiguous row blocks balancing nnz + row_weight*rows (Zipf row lengths)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    m = len(rp) - 1
    cost = rp.astype(np.float64) + row_weight * np.arange(m + 1)
    total = cost[-1]
    bounds = [0]
    for g in range(1, world):
        b = int(np.searchsorted(cost, total * g / world))
        bounds.append(min(max(b, bounds[-1]), m))
    bounds.append(m)
    return [(bounds[g], bounds[g + 1] - bounds[g]) for g in range(world)]


def shard_csr(csr, row0: int, rows: int):
    """Local CSR (rows x n) of global rows [row0, row0+rows), row_ptr rebased to 0."""
    m, n, rp, ci, v = csr
    e0, e1 = int(rp[row0]), int(rp[row0 + rows])
    return rows, n, (np.asarray(rp[row0:row0 + rows + 1]) - e0).astype(np.int64), ci[e0:e1], v[e0:e1]


def shard_dense(a: np.ndarray, row0: int, rows: int) -> np.ndarray:
    return np.asfortranarray(a[row0:row0 + rows])


def nccl_bootstrap(rank: int, group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id; torch.distributed broadcasts it."""
    import torch.distributed as dist

    from .qbfac import Context

    obj = [Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def sharded_context(device: int):
    """Context for this rank of the current torch.distributed world (NCCL communicator)."""
    import torch.distributed as dist

    from .qbfac import Context

    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return Context(device)
    return Context(device, rank, world, nccl_bootstrap(rank))
