"""Multi-rank plumbing: one process per GPU, torch.distributed only for the host-side
handshake (CUDA IPC handle / NCCL id exchange, barriers, max-over-ranks timing).  The halo data
itself moves GPU-to-GPU inside the library (hg_dmp_run): NVLink peer stores fused into the
stencil kernel (transport "p2p"), or NCCL send/recv driven from C++ (transport "nccl")."""
from __future__ import annotations

from typing import List, Sequence

from . import coord_from_rank, neighbor_rank


def face_neighbors(rank: int, grid: Sequence[int]) -> List[int]:
    """Ranks one step away along each grid dimension (no wrap, dmp_ops.cpp:39-49)."""
    out = []
    for d in range(len(grid)):
        for s in (-1, 1):
            dirv = [0] * len(grid)
            dirv[d] = s
            n = neighbor_rank(rank, dirv, grid)
            if n >= 0 and n not in out:
                out.append(n)
    return out


def weak_grid(world: int, ndim: int = 3) -> List[int]:
    """Slabs along dim 0: faces are contiguous planes, <= 2 neighbours per rank."""
    return [world] + [1] * (ndim - 1)


def strong_grid(world: int) -> List[int]:
    """Process grids (z, y, x) for a fixed global domain that keep x, the contiguous dim,
    whole: 1, 2x1x1, 2x2x1, 2x4x1.  Grids splitting x work (packed slabs on the fused path)
    but ran 11% slower at N=4 (1x2x2 2439 vs 2x2x1 2739 GPts/s); rank shapes with x = 2048 and
    y = 512 ran fastest alone (profiles/r2_geo_ab.log)."""
    table = {1: [1, 1, 1], 2: [2, 1, 1], 4: [2, 2, 1], 8: [2, 4, 1]}
    if world in table:
        return table[world]
    return weak_grid(world)


def connect(dmp, rank: int, grid: Sequence[int], world: int, group=None) -> List[int]:
    """All-gather every rank's IPC blob; import those of the face neighbours."""
    import torch.distributed as dist
    blobs = [None] * world
    dist.all_gather_object(blobs, dmp.export(), group=group)
    nbrs = face_neighbors(rank, grid)
    for r in nbrs:
        dmp.import_peer(r, blobs[r])
    return nbrs


def origin_of(rank: int, grid: Sequence[int], core: Sequence[int]) -> List[int]:
    """Global logical offset of a rank's local buffers (scatterRank, simulator.cpp:995-1025)."""
    c = coord_from_rank(rank, grid)
    return [c[d] * core[d] for d in range(len(grid))]


def make_dmp(plan, decomp, rank: int, grid: Sequence[int], world: int, transport: str = "p2p",
             timeout_s: float = 0.0, depth: int = 1, group=None):
    """This rank's hg_dmp on the chosen transport, connected: P2P ranks exchange CUDA IPC
    blobs with their face neighbours; NCCL ranks share one ncclUniqueId (rank 0's)."""
    import torch.distributed as dist

    from . import Dmp, nccl_unique_id
    if transport == "nccl":
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        return Dmp(plan, decomp, rank, transport="nccl", nccl_id=box[0], nranks=world,
                   timeout_s=timeout_s, depth=depth)
    dmp = Dmp(plan, decomp, rank, timeout_s=timeout_s, depth=depth)
    connect(dmp, rank, grid, world, group=group)
    return dmp
