"""Multi-rank plumbing: one process per GPU, torch.distributed only for the host-side
handshake (CUDA IPC handle exchange, barriers, max-over-ranks timing).  The halo data itself
moves GPU-to-GPU over NVLink through the dmp put kernels (hg_dmp_run)."""
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
    """Near-cubic process grids for a fixed global domain (1, 2x1x1, 2x2x1, 2x2x2)."""
    table = {1: [1, 1, 1], 2: [2, 1, 1], 4: [2, 2, 1], 8: [2, 2, 2]}
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


class NcclSwap:
    """The comparison transport (SURVEY §8 e): every dmp.swap of a step as packed boxes moved
    by NCCL point-to-point (torch.distributed batch_isend_irecv), then unpacked -- the
    reference's RankHooks::swap (simulator.cpp:772-834) with NCCL as the Transport.  The
    product path is hg_dmp_run (the stencil kernel stores the next step's send boxes straight
    into the neighbours' halos over NVLink); this class exists to measure against it.

    One step = for each swap in program order: pack every send box (hg_plan_pack), one NCCL
    group of sends/receives with the face neighbours, unpack into the halo boxes; then the
    stencil step (hg_plan_run(1)).  Same stream throughout; NCCL waits on it and it waits on
    NCCL (work.wait())."""

    def __init__(self, plan, decomp, rank: int, grid: Sequence[int], stream=None):
        import numpy as np
        import torch
        self.plan, self.rank, self.stream = plan, rank, stream
        n = decomp.ndim
        self.dtype = torch.float32 if plan.program.dtype == np.float32 else torch.float64
        dev = torch.device("cuda", torch.cuda.current_device())
        self.swaps = []
        for s in range(decomp.nswaps):
            sw = decomp.swaps[s]
            jobs = []
            for k in range(sw.nexchanges):
                e = sw.ex[k]
                to = list(e.to[:n])
                nb = neighbor_rank(rank, to, grid)
                if nb < 0:
                    continue
                size = list(e.size[:n])
                cnt = 1
                for x in size:
                    cnt *= x
                src_at = [e.at[d] + e.offset[d] for d in range(n)]
                jobs.append((nb, src_at, list(e.at[:n]), size,
                             torch.empty(cnt, dtype=self.dtype, device=dev),
                             torch.empty(cnt, dtype=self.dtype, device=dev)))
            self.swaps.append((sw.field, jobs))
        self.bytes = 0

    def step(self):
        import torch.distributed as dist
        perm, _ = self.plan.binding()
        for field, jobs in self.swaps:
            if not jobs:
                continue
            b = perm[field]
            ops = []
            for nb, src_at, dst_at, size, sbuf, rbuf in jobs:
                self.plan.pack(b, src_at, size, sbuf.data_ptr(), self.stream)
                ops.append(dist.P2POp(dist.isend, sbuf, nb))
                ops.append(dist.P2POp(dist.irecv, rbuf, nb))
                self.bytes += sbuf.numel() * sbuf.element_size()
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for nb, src_at, dst_at, size, sbuf, rbuf in jobs:
                self.plan.unpack(b, dst_at, size, rbuf.data_ptr(), self.stream)
        self.plan.run(1, stream=self.stream)

    def run(self, steps: int):
        for _ in range(steps):
            self.step()
