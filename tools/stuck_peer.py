"""Stuck-peer detection check (launched by tests/test_multigpu.py via torchrun, 2 ranks).

Rank 1 connects its dmp but never runs a step.  Rank 0 runs: its standalone put goes out, its
stencil's halo-reading CTAs wait for rank 1's round, which never comes.  The waits are bounded
(2 s here), so instead of hanging the GPU the run records the timeout and hg_dmp_status raises
HG_ETRAP naming the rank, the face and the epoch -- the GPU counterpart of the reference's
deadlock report (simulator.cpp:143-173, 1174-1187).  Later calls fail fast with the same error.
"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402
from paper_2404_02218_b200 import dist as hd  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 64, 4, "f32"))
    local, dc = prog.decompose([2, 1, 1])
    plan = hg.Plan(local, int(os.environ["LOCAL_RANK"]))
    plan.init_fields(origin=hd.origin_of(rank, [2, 1, 1], list(dc.core[:3])))
    dmp = hd.make_dmp(plan, dc, rank, [2, 1, 1], world, timeout_s=2.0)
    dist.barrier()
    ok = True
    if rank == 0:
        t0 = time.time()
        dmp.run(3)
        try:
            dmp.status()
            ok = False
            print("no error reported", flush=True)
        except hg.HgError as e:
            msg = str(e)
            print(f"rank 0 after {time.time() - t0:.1f} s: {msg}", flush=True)
            ok = "did not arrive" in msg and "rank 1" in msg
        try:  # sticky: the next call fails fast
            dmp.run(1)
            ok = False
        except hg.HgError:
            pass
        if ok:
            print("STUCK-PEER REPORTED", flush=True)
    dist.barrier()  # rank 1 keeps its buffers mapped until rank 0 is done
    dmp.close()
    plan.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
