"""Multi-process dmp check (one rank per GPU, CUDA IPC + NVLink puts): after T steps every
rank's local buffers (cores AND halos) must equal the oracle's restatement of the reference's
RankHooks::swap loop bit for bit.  Launched by tests/test_multigpu.py via torchrun."""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="heat")
    ap.add_argument("--rank", type=int, default=3)
    ap.add_argument("--extent", type=int, default=48)
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--grid", default=None)
    ap.add_argument("--extents", default=None,
                    help="global core extents AxBxC (non-cubic; overrides --extent)")
    ap.add_argument("--T", type=int, default=5)
    ap.add_argument("--calls", default=None, help="split T over several run calls, e.g. 2,3")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="p2p: fused NVLink puts; nccl: packed boxes over NCCL (C++ transport)")
    ap.add_argument("--upload", action="store_true",
                    help="the e2e path of bench.py: fields from pinned host buffers via "
                         "hg_plan_upload_live over poisoned device buffers")
    ap.add_argument("--depth", type=int, default=1,
                    help="deep halos: exchange every DEPTH steps (cores checked against the "
                         "oracle's serial run of the global program)")
    ap.add_argument("--golden", default=None,
                    help="a decomposed_authored program of tests/golden (multi-apply)")
    a = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    lr = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr)
    dist.init_process_group("gloo")
    grid = [int(x) for x in a.grid.split("x")] if a.grid else [world] + [1] * (a.rank - 1)
    if a.golden:
        import json
        with open(os.path.join(REPO, "tests", "golden", "reference_golden.json")) as f:
            (case,) = [c for c in json.load(f)["decomposed_authored"] if c["name"] == a.golden]
        prog = hg.Program.from_json(case["program"])
        a.rank = prog.rank
        grid = [int(x) for x in a.grid.split("x")] if a.grid else case["grid"]
    else:
        prog = hg.build_kernel(hg.KernelSpec(a.kind, a.rank, a.extent, a.order, "f32"))
        if a.extents:
            prog = prog.with_extents([int(x) for x in a.extents.split("x")])
    local, dc = prog.decompose(grid, depth=a.depth)
    plan = hg.Plan(local, lr)
    coord = hg.coord_from_rank(rank, grid)
    plan.init_fields(origin=[coord[d] * dc.core[d] for d in range(a.rank)])
    from paper_2404_02218_b200 import dist as hd
    dmp = hd.make_dmp(plan, dc, rank, grid, world, transport=a.transport, depth=a.depth)
    dist.barrier()
    if a.upload:
        host = [torch.from_numpy(plan.download(i)).pin_memory().numpy()
                for i in range(local.nfields)]
        for i in range(local.nfields):  # poison: a skipped region that mattered would show
            plan.upload(i, np.full_like(host[i], np.float32(1e30)))
        plan.reset_binding()
        for i in range(local.nfields):
            plan.upload(i, host[i], live=True)
        dmp.invalidate()  # collective: the next run starts with the receiver-ready handshake
    calls = [int(x) for x in a.calls.split(",")] if a.calls else [a.T]
    assert sum(calls) == a.T
    for c in calls:
        dmp.run(c)
    dmp.status()
    torch.cuda.synchronize()
    perm, _ = plan.binding()
    got = [plan.download(p) for p in perm]
    from oracle import Port
    port = Port()
    glob = port.initial_fields(prog)
    lbs = [prog.field_bounds(i)[0] for i in range(prog.nfields)]
    if a.depth > 1:
        # deep halos: local buffers are wider than the reference's; the cores (what simulate
        # gathers) must equal the serial run of the global program bit for bit
        perm_o = port.run(prog, glob, a.T)
        ok = perm == perm_o
        sr = local.store_region(0)
        for i, g in enumerate(got):
            llo = local.field_bounds(perm[i])[0]
            glo = lbs[perm_o[i]]
            src = tuple(slice(sr.lb[d] - llo[d], sr.ub[d] - llo[d]) for d in range(a.rank))
            dst = tuple(slice(sr.lb[d] + coord[d] * dc.core[d] - glo[d],
                              sr.ub[d] + coord[d] * dc.core[d] - glo[d]) for d in range(a.rank))
            ok = ok and np.array_equal(g[src].view(np.uint8), glob[perm_o[i]][dst].view(np.uint8))
    else:
        want = port.simulate_rank_state(local, dc, glob, lbs, a.T, rank)
        ok = all(np.array_equal(g.view(np.uint8), w.view(np.uint8)) for g, w in zip(got, want))
    flag = torch.tensor([0 if ok else 1])
    dist.all_reduce(flag)
    dist.barrier()
    dmp.close()
    plan.close()
    if rank == 0:
        print(f"dmp_check {a.kind}{a.rank}d n{a.extent} o{a.order} grid={grid} T={a.T} "
              f"transport={a.transport} depth={a.depth}: {'OK' if flag.item() == 0 else 'MISMATCH'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
