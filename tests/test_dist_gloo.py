"""Host side of the multi-rank protocol on CPU (gloo, world_size 2 and 4): each rank imports
exactly its face neighbours' IPC blobs, and the per-rank geometry (grid, origin, neighbours)
matches the reference's decomposition arithmetic."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeDmp:
    def __init__(self, rank):
        self.rank = rank
        self.imported = {}

    def export(self):
        return f"blob-of-{self.rank}".encode()

    def import_peer(self, r, blob):
        self.imported[r] = blob


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, grid, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_02218_b200 import dist as hd
    d = FakeDmp(rank)
    nbrs = hd.connect(d, rank, grid, world)
    origin = hd.origin_of(rank, grid, [8, 8, 8])
    dist.barrier()
    q.put((rank, sorted(nbrs), {k: v.decode() for k, v in d.imported.items()}, origin))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,grid", [(2, [2, 1, 1]), (4, [2, 2, 1]), (4, [4, 1, 1])])
def test_handle_exchange(world, grid):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, nbrs, imported, origin = q.get(timeout=120)
        res[r] = (nbrs, imported, origin)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import paper_2404_02218_b200 as hg
    for r, (nbrs, imported, origin) in res.items():
        want = set()
        for d in range(3):
            for s in (-1, 1):
                dv = [0, 0, 0]
                dv[d] = s
                n = hg.neighbor_rank(r, dv, grid)
                if n >= 0:
                    want.add(n)
        assert set(nbrs) == want
        assert imported == {n: f"blob-of-{n}" for n in want}
        c = hg.coord_from_rank(r, grid)
        assert origin == [c[d] * 8 for d in range(3)]


def test_grids():
    from paper_2404_02218_b200 import dist as hd
    assert hd.weak_grid(8) == [8, 1, 1]
    assert hd.strong_grid(8) == [2, 4, 1] and hd.strong_grid(4) == [2, 2, 1]
    assert hd.face_neighbors(0, [2, 2, 2]) == [4, 2, 1]
